// radix_sort.cuh -- stable LSD radix sort of (u64 key, i32 value) pairs on the
// device: north-star kernel 2 ("a stable radix sort ... on the priority key
// orders the queues, with tie-breaks identical to the reference").
//
// The reference orders the waiting queue by (priority, arrival, rel_id)
// (engine.py:175-176, 277-281).  Keys here are okey(priority) (an
// order-preserving map of the double, engine_state.cuh) and values admission
// ranks, which are sorted by (arrival, rel_id) (engine.py:211-213): sorting
// pairs that start in rank order *stably* by key yields exactly the
// reference's order.  Used for
//   * the static waiting order at engine creation (the first-sight / sp
//     priorities of every relQuery, engine.cu build_trace), and
//   * parity mode's full per-iteration waiting order (rs_engine_read_order):
//     (iteration row, key, rank) triples sorted by key, then stably by row.
//
// Eight 8-bit digits, least significant first; a pass whose digit is the same
// for every key is skipped (priorities of one trace share their exponent
// bits).  Each pass: per-tile digit histograms, an exclusive scan in
// (digit, tile) order, and a stable scatter that ranks each 1024-key chunk with
// __match_any_sync per warp plus a per-digit scan over the warps.  Small
// inputs (<= kSortOneCta keys) run every pass inside one CTA, one launch;
// larger ones run each pass as three grid launches over kSortTile-key tiles,
// stream-ordered with no host round trip (sort_pairs_enqueue): the identity
// passes are recognised on the device from the all-pass digit histogram.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rsd {

constexpr int kSortThreads = 1024;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortOneCta = 4096;  // one-CTA sort up to this many keys (its passes run serially on one SM)
constexpr int kSortTile = 2 * kSortThreads;  // keys per CTA tile of the multi-CTA passes

struct SortChunkSmem {
  unsigned wcnt[kSortWarps][256];  // per-warp digit counts -> per-warp digit offsets
  unsigned base[256];              // running output position per digit (this CTA's share)
  unsigned hist[256];
  int same;
};

__device__ __forceinline__ unsigned sort_digit(unsigned long long k, int shift) {
  return (unsigned)(k >> shift) & 0xFFu;
}

// One count per key of digit d (d >= 256: no key) into h, one shared-memory
// atomic per distinct digit of the warp (all 32 lanes must call it).
__device__ __forceinline__ void hist_add(unsigned* h, unsigned d) {
  const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
  if (d < 256u && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[d], (unsigned)__popc(peers));
}

// Histogram of digit `shift` over keys [lo, hi) into sm.hist (zeroed here).
__device__ __forceinline__ void sort_hist(const unsigned long long* keys, long long lo, long long hi, int shift,
                                          SortChunkSmem& sm) {
  for (int b = threadIdx.x; b < 256; b += kSortThreads) sm.hist[b] = 0;
  __syncthreads();
  for (long long c0 = lo; c0 < hi; c0 += kSortThreads) {  // warp-uniform trip count
    const long long i = c0 + threadIdx.x;
    hist_add(sm.hist, i < hi ? sort_digit(keys[i], shift) : 256u + (threadIdx.x & 31));
  }
  __syncthreads();
}

// Stable scatter of [lo, hi) by digit `shift`: sm.base[d] holds the first
// output position of this range's keys with digit d (advanced here).
__device__ __forceinline__ void sort_scatter(const unsigned long long* sk, const int* sv, unsigned long long* dk,
                                             int* dv, long long lo, long long hi, int shift, SortChunkSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (long long c0 = lo; c0 < hi; c0 += kSortThreads) {
    const long long i = c0 + threadIdx.x;
    const bool in = i < hi;
    unsigned long long k = 0;
    int v = 0;
    unsigned d = 256u + (unsigned)lane;  // out-of-range lanes: a group of their own
    if (in) {
      k = sk[i];
      v = sv[i];
      d = sort_digit(k, shift);
    }
#pragma unroll
    for (int b = lane; b < 256; b += 32) sm.wcnt[warp][b] = 0;
    __syncwarp();
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
    const unsigned rank = __popc(peers & lt);
    if (in && rank == 0) sm.wcnt[warp][d] = __popc(peers);
    __syncthreads();
    // per digit: exclusive scan over the warps, from the digit's running base --
    // four threads per digit (the same warp), eight warps' counts each
    {
      static_assert(kSortThreads == 4 * 256 && kSortWarps == 32, "4 threads x 8 warps per digit");
      const int d = threadIdx.x >> 2, part = threadIdx.x & 3;
      unsigned c8[8], sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c8[i] = sm.wcnt[part * 8 + i][d];
        sum += c8[i];
      }
      unsigned incl = sum;
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        const unsigned x = __shfl_up_sync(0xFFFFFFFFu, incl, o, 4);
        if (part >= o) incl += x;
      }
      unsigned run = sm.base[d] + incl - sum;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        sm.wcnt[part * 8 + i][d] = run;
        run += c8[i];
      }
      __syncwarp();
      if (part == 3) sm.base[d] = run;  // every part has read the base
    }
    __syncthreads();
    if (in) {
      const unsigned pos = sm.wcnt[warp][d] + rank;
      dk[pos] = k;
      dv[pos] = v;
    }
    __syncthreads();
  }
}

// One CTA sorts n <= kSortOneCta pairs, every pass in this launch; (k0, v0)
// hold the input and receive the result, (k1, v1) are scratch of the same size.
__global__ void __launch_bounds__(kSortThreads, 1)
    sort_pairs_one_cta(unsigned long long* k0, int* v0, unsigned long long* k1, int* v1, int n) {
  __shared__ SortChunkSmem sm;
  unsigned long long *sk = k0, *dk = k1;
  int *sv = v0, *dv = v1;
  for (int shift = 0; shift < 64; shift += 8) {
    sort_hist(sk, 0, n, shift, sm);
    if (threadIdx.x == 0) sm.same = 0;
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += kSortThreads)
      if (sm.hist[b] == (unsigned)n) sm.same = 1;
    __syncthreads();
    if (sm.same) continue;  // every key has this digit: the pass is the identity
    if (threadIdx.x < 32) {  // exclusive scan of the 256 digit counts (8 per lane)
      unsigned c[8], s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = sm.hist[threadIdx.x * 8 + j];
        s += c[j];
      }
      unsigned incl = s;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned o = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if ((int)threadIdx.x >= d) incl += o;
      }
      unsigned run = incl - s;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        sm.base[threadIdx.x * 8 + j] = run;
        run += c[j];
      }
    }
    __syncthreads();
    sort_scatter(sk, sv, dk, dv, 0, n, shift, sm);
    unsigned long long* tk = sk;
    sk = dk;
    dk = tk;
    int* tv = sv;
    sv = dv;
    dv = tv;
  }
  if (sk != k0) {  // an odd number of passes ran: the result is in the scratch pair
    for (int i = threadIdx.x; i < n; i += kSortThreads) {
      k0[i] = sk[i];
      v0[i] = sv[i];
    }
  }
}

// Multi-CTA passes (large inputs).  1. digit histograms of every pass over
// all keys (which passes are not the identity), 2. per pass: tile histograms
// (digit-major: th[d * n_tiles + tile]), 3. one-CTA exclusive scan of them,
// 4. stable scatter of each tile from its scanned bases.
__global__ void __launch_bounds__(kSortThreads) sort_global_hist(const unsigned long long* keys, long long n,
                                                                 unsigned long long* hist /* [8][256] */) {
  __shared__ unsigned h[8][256];
  for (int b = threadIdx.x; b < 8 * 256; b += kSortThreads) (&h[0][0])[b] = 0;
  __syncthreads();
  for (long long c0 = (long long)blockIdx.x * kSortThreads; c0 < n; c0 += (long long)gridDim.x * kSortThreads) {
    const long long i = c0 + threadIdx.x;  // warp-uniform trip count
    const unsigned long long k = i < n ? keys[i] : 0ULL;
#pragma unroll
    for (int p = 0; p < 8; ++p) hist_add(h[p], i < n ? sort_digit(k, 8 * p) : 256u + (threadIdx.x & 31));
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 8 * 256; b += kSortThreads)
    if ((&h[0][0])[b]) atomicAdd(&hist[b], (unsigned long long)(&h[0][0])[b]);
}

// Pass `shift` is the identity when every key has the same digit there: the
// count of any one key's digit (keys[0]'s) is n.  gh = sort_global_hist's counts.
__device__ __forceinline__ bool sort_identity(const unsigned long long* keys, long long n, int shift,
                                              const unsigned long long* gh) {
  return gh[(shift >> 3) * 256 + sort_digit(keys[0], shift)] == (unsigned long long)n;
}

__global__ void __launch_bounds__(kSortThreads) sort_tile_hist(const unsigned long long* keys, long long n, int shift,
                                                               unsigned* th, int n_tiles, const unsigned long long* gh) {
  if (gh && sort_identity(keys, n, shift, gh)) return;
  __shared__ SortChunkSmem sm;
  const long long lo = (long long)blockIdx.x * kSortTile;
  const long long hi = lo + kSortTile < n ? lo + kSortTile : n;
  sort_hist(keys, lo, hi, shift, sm);
  for (int b = threadIdx.x; b < 256; b += kSortThreads) th[(long long)b * n_tiles + blockIdx.x] = sm.hist[b];
}

__global__ void __launch_bounds__(kSortThreads) sort_scan(unsigned* th, long long m, const unsigned long long* keys,
                                                          long long n, int shift, const unsigned long long* gh) {
  if (gh && sort_identity(keys, n, shift, gh)) return;
  __shared__ unsigned wsum[kSortWarps];
  __shared__ unsigned carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (long long c0 = 0; c0 < m; c0 += kSortThreads) {
    const long long i = c0 + threadIdx.x;
    const unsigned x = i < m ? th[i] : 0u;
    unsigned incl = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned o = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += o;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    unsigned before = carry, total = 0;
    for (int w = 0; w < kSortWarps; ++w) {
      const unsigned t = wsum[w];
      if (w < warp) before += t;
      total += t;
    }
    if (i < m) th[i] = before + incl - x;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSortThreads) sort_tile_scatter(const unsigned long long* sk, const int* sv,
                                                                  unsigned long long* dk, int* dv, long long n,
                                                                  int shift, const unsigned* th, int n_tiles,
                                                                  const unsigned long long* gh) {
  __shared__ SortChunkSmem sm;
  const long long lo = (long long)blockIdx.x * kSortTile;
  const long long hi = lo + kSortTile < n ? lo + kSortTile : n;
  if (gh && sort_identity(sk, n, shift, gh)) {  // the identity pass: the tile as it is (keeps the ping-pong fixed)
    for (long long i = lo + threadIdx.x; i < hi; i += kSortThreads) {
      dk[i] = sk[i];
      dv[i] = sv[i];
    }
    return;
  }
  for (int b = threadIdx.x; b < 256; b += kSortThreads) sm.base[b] = th[(long long)b * n_tiles + blockIdx.x];
  __syncthreads();
  sort_scatter(sk, sv, dk, dv, lo, hi, shift, sm);
}

// The grid passes, enqueued on `st` with no host round trip: all eight digits
// run (identity passes copy), so the sorted pairs end in (k, v).  Scratch:
// (k1, v1) n pairs, gh 8 * 256 counts, th 256 * ceil(n / kSortTile) counts.
inline cudaError_t sort_pairs_enqueue(unsigned long long* k, int* v, unsigned long long* k1, int* v1,
                                      unsigned long long* gh, unsigned* th, long long n, cudaStream_t st) {
  const long long tiles = (n + kSortTile - 1) / kSortTile;
  cudaError_t e = cudaMemsetAsync(gh, 0, 8 * 256 * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  sort_global_hist<<<(unsigned)(tiles < 148 ? tiles : 148), kSortThreads, 0, st>>>(k, n, gh);
  unsigned long long *sk = k, *dk = k1;
  int *sv = v, *dv = v1;
  for (int p = 0; p < 8; ++p) {
    sort_tile_hist<<<(unsigned)tiles, kSortThreads, 0, st>>>(sk, n, 8 * p, th, (int)tiles, gh);
    sort_scan<<<1, kSortThreads, 0, st>>>(th, 256 * tiles, sk, n, 8 * p, gh);
    sort_tile_scatter<<<(unsigned)tiles, kSortThreads, 0, st>>>(sk, sv, dk, dv, n, 8 * p, th, (int)tiles, gh);
    unsigned long long* tk = sk;
    sk = dk;
    dk = tk;
    int* tv = sv;
    sv = dv;
    dv = tv;
  }
  return cudaGetLastError();
}

}  // namespace rsd
