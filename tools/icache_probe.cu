// icache_probe.cu -- cost of one PCG64 128-bit step + output on warp 0 in a
// tiny kernel (warm I-cache) vs inside the engine (tools/README).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2601_11546_b200/csrc/pcg64.cuh"
using namespace rsd;
__global__ void k(long long* out, unsigned long long a, unsigned long long b) {
  __shared__ JumpEntry js[32];
  if (threadIdx.x < 32) { js[threadIdx.x].a = U128{a + threadIdx.x, b}; js[threadIdx.x].c = U128{b, a}; }
  __syncthreads();
  if (threadIdx.x < 32) {
    U128 sb{a, b};
    long long t0 = clock64();
    uint64_t acc = 0;
    for (int i = 0; i < 64; ++i) {
      const U128 st = add128(mul128(js[threadIdx.x].a, sb), js[threadIdx.x].c);
      acc ^= pcg_output(st);
      sb.hi = __shfl_sync(0xffffffffu, st.hi, 31);
      sb.lo = __shfl_sync(0xffffffffu, st.lo, 31);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0) / 64; out[1] = acc; }
  }
}
int main() { long long* o; cudaMalloc(&o, 16); k<<<1, 512>>>(o, 3, 5); k<<<1, 512>>>(o, 3, 5); long long r[2];
  cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost); printf("{\"pcg_step_plus_shfl_cycles\": %lld}\n", r[0]); }
