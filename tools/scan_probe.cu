// scan_probe.cu -- cost of block-scan variants (512 threads, one CTA).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2601_11546_b200/csrc/block.cuh"
using namespace rsd;

struct Sm32 { int w[4][kWarps]; int tot[4]; };

template <int N>
__device__ __forceinline__ void scan32(int (&v)[N], Sm32& sm, int (&tot)[N]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < N; ++c) v[c] = warp_incl_scan(v[c]);
  if (lane == 31) {
#pragma unroll
    for (int c = 0; c < N; ++c) sm.w[c][warp] = v[c];
  }
  __syncthreads();
  // every warp scans the 16 warp totals itself (no second barrier round)
#pragma unroll
  for (int c = 0; c < N; ++c) {
    int x = lane < kWarps ? sm.w[c][lane] : 0;
    x = warp_incl_scan(x);
    const int before = __shfl_sync(kFull, x, (warp + 31) & 31);
    tot[c] = __shfl_sync(kFull, x, kWarps - 1);
    if (warp > 0) v[c] += before;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(512, 1) probe(long long* out) {
  __shared__ ScanSmem scan;
  __shared__ Sm32 s32;
  long long acc = 0;
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < 128; ++i) { long long v[2] = {threadIdx.x + i, 1}, tot[2]; block_incl_scan<2>(v, scan, tot); acc += v[0] + tot[1]; }
  t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / 128;
  t0 = clock64();
  for (int i = 0; i < 128; ++i) { long long v[1] = {threadIdx.x + i}, tot[1]; block_incl_scan<1>(v, scan, tot); acc += v[0] + tot[0]; }
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / 128;
  t0 = clock64();
  for (int i = 0; i < 128; ++i) { int v[2] = {(int)threadIdx.x + i, 1}, tot[2]; scan32<2>(v, s32, tot); acc += v[0] + tot[1]; }
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / 128;
  t0 = clock64();
  for (int i = 0; i < 128; ++i) { int v[1] = {(int)threadIdx.x + i}, tot[1]; scan32<1>(v, s32, tot); acc += v[0] + tot[0]; }
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / 128;
  // warp-only scan of 32 ints
  if (threadIdx.x < 32) {
    int x = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < 128; ++i) x = warp_incl_scan(x + i) & 0xFFFF;
    t1 = clock64();
    if (threadIdx.x == 0) out[4] = (t1 - t0) / 128;
    acc += x;
  }
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < 128; ++i) { long long s = block_sum((long long)threadIdx.x + i, scan); acc += s; }
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0) / 128;
  if (threadIdx.x == 7) out[9] = acc;
}
int main() {
  long long* o; cudaMalloc(&o, 16 * 8);
  probe<<<1, 512>>>(o); probe<<<1, 512>>>(o);
  long long r[16]; cudaMemcpy(r, o, sizeof r, cudaMemcpyDeviceToHost);
  printf("{\"scan64x2\": %lld, \"scan64x1\": %lld, \"scan32x2_2sync\": %lld, \"scan32x1_2sync\": %lld, \"warp_scan32\": %lld, \"block_sum64\": %lld}\n", r[0], r[1], r[2], r[3], r[4], r[5]);
}
