// lat_probe2.cu -- B200 latencies the scheduler's serial chains are made of:
// dependent fp64 add / mul (__dadd_rn/__dmul_rn), fp64 divide, a dependent
// shared-memory load through a shared vs a generic pointer, and a warp
// shuffle.  One thread, clock64 around 256-long dependent chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o lat_probe2 lat_probe2.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* out, double x, double y, int* gidx) {
  __shared__ int sidx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sidx[i] = (i * 7 + 3) & 1023;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double a = x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) a = __dadd_rn(a, y);
  long long t1 = clock64();
  double m = x;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) m = __dmul_rn(m, y);
  long long t2 = clock64();
  double d = x;
#pragma unroll 1
  for (int i = 0; i < 64; ++i) d = __ddiv_rn(y, d + 1.0);
  long long t3 = clock64();
  int p = 0;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) p = sidx[p];
  long long t4 = clock64();
  volatile int* gp = (volatile int*)(void*)sidx;  // generic pointer to shared memory
  int* g = (int*)gp;
  int q = 0;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) q = g[q];
  long long t5 = clock64();
  out[0] = (t1 - t0) / 256;
  out[1] = (t2 - t1) / 256;
  out[2] = (t3 - t2) / 64;
  out[3] = (t4 - t3) / 256;
  out[4] = (t5 - t4) / 256;
  out[5] = (long long)(a + m + d) + p + q;
}
__global__ void kshfl(long long* out) {
  int v = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / 256; out[1] = v; }
}
int main() {
  long long* o;
  cudaMalloc(&o, 64);
  long long r[8];
  k<<<1, 128>>>(o, 1.000001, 1.0000001, nullptr);
  k<<<1, 128>>>(o, 1.000001, 1.0000001, nullptr);
  cudaMemcpy(r, o, 48, cudaMemcpyDeviceToHost);
  printf("{\"dadd\": %lld, \"dmul\": %lld, \"ddiv\": %lld, \"lds_dep\": %lld, \"ld_generic_smem_dep\": %lld}\n", r[0], r[1],
         r[2], r[3], r[4]);
  kshfl<<<1, 32>>>(o);
  kshfl<<<1, 32>>>(o);
  cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
  printf("{\"shfl_dep\": %lld}\n", r[0]);
}
