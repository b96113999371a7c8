// latency_probe.cu -- one-off calibration of the costs the scheduler's
// critical path is made of (single-CTA, 512 threads): dependent L2 loads,
// smem loads, __syncthreads, a 3-sync block scan, fp64 add chains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/latency_probe tools/latency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2601_11546_b200/csrc/block.cuh"
using namespace rsd;

__global__ void __launch_bounds__(512, 1) probe(int* buf, int n, long long* out) {
  __shared__ int sm[4096];
  __shared__ ScanSmem scan;
  for (int i = threadIdx.x; i < 4096; i += 512) sm[i] = (i * 7 + 3) & 4095;
  __syncthreads();
  long long t0, t1;
  // 1. dependent global loads (pointer chase), thread 0
  if (threadIdx.x == 0) {
    int p = 0;
    for (int i = 0; i < 64; ++i) p = buf[p];  // warm
    t0 = clock64();
    for (int i = 0; i < 256; ++i) p = buf[p];
    t1 = clock64();
    out[0] = (t1 - t0) / 256;
    out[9] = p;
    // 2. dependent smem loads
    int q = 0;
    t0 = clock64();
    for (int i = 0; i < 1024; ++i) q = sm[q];
    t1 = clock64();
    out[1] = (t1 - t0) / 1024;
    out[10] = q;
    // 5. fp64 add chain
    double d = 1.0;
    t0 = clock64();
    for (int i = 0; i < 1024; ++i) d = __dadd_rn(d, 1e-9);
    t1 = clock64();
    out[4] = (t1 - t0) / 1024;
    out[11] = (long long)d;
  }
  __syncthreads();
  // 3. __syncthreads
  t0 = clock64();
  for (int i = 0; i < 256; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / 256;
  // 4. 2-component block scan
  long long acc = 0;
  t0 = clock64();
  for (int i = 0; i < 128; ++i) {
    long long v[2] = {threadIdx.x + i, 1}, tot[2];
    block_incl_scan<2>(v, scan, tot);
    acc += v[0] + tot[1];
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / 128;
  // 6. thread 0 global store then other threads read after sync
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < 64; ++i) {
    if (threadIdx.x == 0) buf[n + 1] = i;
    __syncthreads();
    acc += buf[n + 1];
    __syncthreads();
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0) / 64;
  // 7. ballot+ffs+shfl per warp (warp 0)
  if (threadIdx.x < 32) {
    int x = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < 256; ++i) {
      unsigned m = __ballot_sync(kFull, (x & 7) == (i & 7));
      x = __shfl_sync(kFull, x + __ffs(m), (i + 1) & 31);
    }
    t1 = clock64();
    if (threadIdx.x == 0) { out[6] = (t1 - t0) / 256; out[12] = x; }
  }
  if (threadIdx.x == 5) out[13] = acc;
}

int main() {
  const int n = 1 << 22;
  int* h = new int[n + 2];
  // random cyclic permutation over 16 MB so each hop misses L1
  for (int i = 0; i < n; ++i) h[i] = (int)(((long long)i * 2654435761LL + 12345) % n);
  int* d;
  long long* o;
  cudaMalloc(&d, (n + 2) * 4);
  cudaMalloc(&o, 16 * 8);
  cudaMemcpy(d, h, (n + 2) * 4, cudaMemcpyHostToDevice);
  probe<<<1, 512>>>(d, n, o);
  probe<<<1, 512>>>(d, n, o);
  long long r[16];
  cudaMemcpy(r, o, sizeof r, cudaMemcpyDeviceToHost);
  printf("{\"dep_global_load_cycles\": %lld, \"dep_smem_load_cycles\": %lld, \"syncthreads_512_cycles\": %lld, "
         "\"block_scan2_cycles\": %lld, \"dadd_chain_cycles\": %lld, \"store_sync_load_sync_cycles\": %lld, "
         "\"ballot_ffs_shfl_cycles\": %lld}\n", r[0], r[1], r[2], r[3], r[4], r[5], r[6]);
  return 0;
}
