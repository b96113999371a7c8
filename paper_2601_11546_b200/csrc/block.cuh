// block.cuh -- CTA-wide scan / reduction primitives (warp shuffles + one smem
// slot per warp).  All threads of the CTA must call them.
#pragma once
#include <stdint.h>

namespace rsd {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xFFFFFFFFu;

// Warp index the compiler cannot relate to threadIdx.x.  Without it, nvcc
// jump-threads an `if (threadIdx.x == 0) {...}` straight into a following
// `if (warp == 0) {...}` body without a reconvergence point, and warp 0 then
// runs the whole warp-specialised section twice (lane 0, then lanes 1-31).
__device__ __forceinline__ int opaque_warp() {
  unsigned t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return (int)(t >> 5);
}

// Lane index with the same property: conditions on it cannot be related to
// threadIdx.x (or to each other) at compile time, so lane-0-only blocks end at
// a reconvergence point before the next warp-wide shuffle / ballot.
__device__ __forceinline__ int opaque_lane() {
  unsigned l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return (int)l;
}

// Stable in-place compaction of list[0, n) to the entries x with keep(x), by
// one whole warp, 32 entries per round; returns the new length (every lane).
// Each round's entries are all read (the ballot) before any is written, and
// writes land below the round's end, so later rounds read unmoved entries.
template <class F>
__device__ __forceinline__ int warp_compact(int* list, const int n, F keep) {
  const int lane = threadIdx.x & 31;
  int w = 0;
#pragma unroll 1
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    int x = 0;
    bool k = false;
    if (i < n) {
      x = list[i];
      k = keep(x);
    }
    const unsigned m = __ballot_sync(kFull, k);
    if (k) list[w + __popc(m & ((1u << lane) - 1u))] = x;
    w += __popc(m);
  }
  __syncwarp();
  return w;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// 32-bit: the shuffle's own in-range predicate guards the add (two
// instructions per step, no lane compares) -- the scans are the largest
// block of hot code in the scheduler iteration.
template <>
__device__ __forceinline__ int warp_incl_scan<int>(int v) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1)
    asm("{\n\t.reg .b32 o;\n\t.reg .pred p;\n\t"
        "shfl.sync.up.b32 o|p, %0, %1, 0, -1;\n\t"
        "@p add.s32 %0, %0, o;\n\t}"
        : "+r"(v)
        : "r"(d));
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    T o = __shfl_xor_sync(kFull, v, d);
    v = o > v ? o : v;
  }
  return v;
}

// Scratch for block scans of up to 4 lanes of int64.
struct ScanSmem {
  long long w[4][kWarps];
  long long tot[4];
};

// Inclusive block scan of N int64 values per thread-slot (N <= 4); returns
// inclusive prefix in v[], block totals in tot[] (visible after return).
template <int N>
__device__ __forceinline__ void block_incl_scan(long long (&v)[N], ScanSmem& sm, long long (&tot)[N]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < N; ++c) v[c] = warp_incl_scan(v[c]);
  if (lane == 31) {
#pragma unroll
    for (int c = 0; c < N; ++c) sm.w[c][warp] = v[c];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < N; ++c) {
      long long x = lane < kWarps ? sm.w[c][lane] : 0;
      x = warp_incl_scan(x);
      if (lane < kWarps) sm.w[c][lane] = x;
      if (lane == kWarps - 1) sm.tot[c] = x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < N; ++c) {
    if (warp > 0) v[c] += sm.w[c][warp - 1];
    tot[c] = sm.tot[c];
  }
  __syncthreads();
}

__device__ __forceinline__ long long block_sum(long long v, ScanSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sm.w[0][warp] = v;
  __syncthreads();
  if (warp == 0) {
    long long x = lane < kWarps ? sm.w[0][lane] : 0;
    x = warp_sum(x);
    if (lane == 0) sm.tot[0] = x;
  }
  __syncthreads();
  long long r = sm.tot[0];
  __syncthreads();
  return r;
}

// Argmin over (key, idx) pairs: smallest key, ties -> smallest idx.
struct ArgminSmem {
  unsigned long long k[kWarps];
  long long i[kWarps];
  unsigned long long rk;
  long long ri;
};

__device__ __forceinline__ void argmin_merge(unsigned long long& k, long long& i, unsigned long long ok,
                                             long long oi) {
  if (ok < k || (ok == k && oi < i)) {
    k = ok;
    i = oi;
  }
}

__device__ __forceinline__ void block_argmin(unsigned long long& key, long long& idx, ArgminSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    unsigned long long ok = __shfl_xor_sync(kFull, key, d);
    long long oi = __shfl_xor_sync(kFull, idx, d);
    argmin_merge(key, idx, ok, oi);
  }
  if (lane == 0) {
    sm.k[warp] = key;
    sm.i[warp] = idx;
  }
  __syncthreads();
  if (warp == 0) {
    unsigned long long k = lane < kWarps ? sm.k[lane] : ~0ULL;
    long long i = lane < kWarps ? sm.i[lane] : (long long)0x7FFFFFFFFFFFFFFFLL;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      unsigned long long ok = __shfl_xor_sync(kFull, k, d);
      long long oi = __shfl_xor_sync(kFull, i, d);
      argmin_merge(k, i, ok, oi);
    }
    if (lane == 0) {
      sm.rk = k;
      sm.ri = i;
    }
  }
  __syncthreads();
  key = sm.rk;
  idx = sm.ri;
  __syncthreads();
}

}  // namespace rsd

namespace rsd {

// 32-bit block scan with two barriers: every warp derives its offset from the
// per-warp totals itself instead of waiting for warp 0 (measured on B200: ~390
// cycles for one component with a second-level shuffle scan vs ~770 for the
// 64-bit three-barrier scan; the redux.sync second level is ~2.5% faster per
// scheduler iteration again and half the code).
struct Scan32Smem {
  int w[4][kWarps];
};

template <int N>
__device__ __forceinline__ void block_scan32(int (&v)[N], Scan32Smem& sm, int (&tot)[N]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < N; ++c) v[c] = warp_incl_scan(v[c]);
  if (lane == 31) {
#pragma unroll
    for (int c = 0; c < N; ++c) sm.w[c][warp] = v[c];
  }
  __syncthreads();
  // second level by hardware reductions: lane l holds warp l's total; the
  // warps before this one and all warps are two masked redux.sync sums
  // (32-bit wrap-around sums are exact two's-complement sums of ints)
#pragma unroll
  for (int c = 0; c < N; ++c) {
    const unsigned x = lane < kWarps ? (unsigned)sm.w[c][lane] : 0u;
    tot[c] = (int)__reduce_add_sync(kFull, x);
    v[c] += (int)__reduce_add_sync(kFull, lane < warp ? x : 0u);
  }
  __syncthreads();
}

// Fused block reduction: count (sum of int) + argmin over (u64 key, int idx).
struct RedSmem {
  unsigned long long k[kWarps];
  int i[kWarps];
  int n[kWarps];
};

__device__ __forceinline__ void block_count_argmin(int& cnt, unsigned long long& key, int& idx, RedSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long ok = __shfl_xor_sync(kFull, key, d);
    const int oi = __shfl_xor_sync(kFull, idx, d);
    cnt += __shfl_xor_sync(kFull, cnt, d);
    if (ok < key || (ok == key && oi < idx)) {
      key = ok;
      idx = oi;
    }
  }
  if (lane == 0) {
    sm.k[warp] = key;
    sm.i[warp] = idx;
    sm.n[warp] = cnt;
  }
  __syncthreads();
  unsigned long long k = lane < kWarps ? sm.k[lane] : ~0ULL;
  int i = lane < kWarps ? sm.i[lane] : 0x7FFFFFFF;
  int n = lane < kWarps ? sm.n[lane] : 0;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long ok = __shfl_xor_sync(kFull, k, d);
    const int oi = __shfl_xor_sync(kFull, i, d);
    n += __shfl_xor_sync(kFull, n, d);
    if (ok < k || (ok == k && oi < i)) {
      k = ok;
      i = oi;
    }
  }
  key = k;
  idx = i;
  cnt = n;
  __syncthreads();
}

}  // namespace rsd

namespace rsd {

// ---------------------------------------------------------------------------
// Warp groups with their own named barrier (bar.sync id, n): the pipelined
// common-configuration iteration runs the state advance on warps 0-7 (group
// M, barrier 1) while warps 8-15 (group D, barrier 2) compute the next
// iteration's priority update; barrier 0 (__syncthreads) is the whole CTA.
// ---------------------------------------------------------------------------
template <int N, int BAR>
struct Grp {
  static constexpr int kN = N;
  static constexpr int kW = N / 32;
  __device__ __forceinline__ static void sync() {
    if constexpr (BAR == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(N) : "memory");
  }
  // barrier + OR of a predicate over the group
  __device__ __forceinline__ static bool sync_or(bool p) {
    if constexpr (BAR == 0) {
      return __syncthreads_or(p);
    } else {
      int r;
      asm volatile(
          "{\n\t.reg .pred q, o;\n\t"
          "setp.ne.s32 q, %1, 0;\n\t"
          "bar.red.or.pred o, %2, %3, q;\n\t"
          "selp.s32 %0, 1, 0, o;\n\t}"
          : "=r"(r)
          : "r"((int)p), "n"(BAR), "n"(N)
          : "memory");
      return r != 0;
    }
  }
};
using GAll = Grp<kThreads, 0>;
constexpr int kMWarps = 8;                   // group M: warps [0, 8)
constexpr int kDWarps = kWarps - kMWarps;    // group D: warps [8, 16)
using GM = Grp<kMWarps * 32, 1>;
using GD = Grp<kDWarps * 32, 2>;
constexpr int kBarHandoff = 3;  // group D has read the state group M is about to change

__device__ __forceinline__ void handoff_arrive() {  // group D
  asm volatile("bar.arrive %0, %1;" ::"n"(kBarHandoff), "n"(kThreads) : "memory");
}
__device__ __forceinline__ void handoff_wait() {  // group M
  asm volatile("bar.sync %0, %1;" ::"n"(kBarHandoff), "n"(kThreads) : "memory");
}
constexpr int kBarExecDone = 5;  // group M has applied the iteration's action (group D may commit its update)
__device__ __forceinline__ void exec_done_arrive() {  // group M
  asm volatile("bar.arrive %0, %1;" ::"n"(kBarExecDone), "n"(kThreads) : "memory");
}
__device__ __forceinline__ void exec_done_wait() {  // group D
  asm volatile("bar.sync %0, %1;" ::"n"(kBarExecDone), "n"(kThreads) : "memory");
}
constexpr int kBarDecision = 6;  // group M has the candidates (S.head, S.taken): group D may start the update
__device__ __forceinline__ void decision_arrive() {  // group M
  asm volatile("bar.arrive %0, %1;" ::"n"(kBarDecision), "n"(kThreads) : "memory");
}
__device__ __forceinline__ void decision_wait() {  // group D
  asm volatile("bar.sync %0, %1;" ::"n"(kBarDecision), "n"(kThreads) : "memory");
}

// block_count_argmin over the G::kN threads of a group (its warps consecutive from warp 0)
template <class G>
__device__ __forceinline__ void group_count_argmin(int& cnt, unsigned long long& key, int& idx, RedSmem& sm) {
  if constexpr (G::kN == kThreads) {
    block_count_argmin(cnt, key, idx, sm);
  } else {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(kFull, key, d);
      const int oi = __shfl_xor_sync(kFull, idx, d);
      cnt += __shfl_xor_sync(kFull, cnt, d);
      if (ok < key || (ok == key && oi < idx)) {
        key = ok;
        idx = oi;
      }
    }
    if (lane == 0) {
      sm.k[warp] = key;
      sm.i[warp] = idx;
      sm.n[warp] = cnt;
    }
    G::sync();
    unsigned long long k = lane < G::kW ? sm.k[lane] : ~0ULL;
    int i = lane < G::kW ? sm.i[lane] : 0x7FFFFFFF;
    int n = lane < G::kW ? sm.n[lane] : 0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(kFull, k, d);
      const int oi = __shfl_xor_sync(kFull, i, d);
      n += __shfl_xor_sync(kFull, n, d);
      if (ok < k || (ok == k && oi < i)) {
        k = ok;
        i = oi;
      }
    }
    G::sync();
    key = k;
    idx = i;
    cnt = n;
  }
}

// block_scan32 over the G::kN threads of a group (thread index within the group
// = threadIdx.x - base; the group's warps are consecutive)
template <class G, int N>
__device__ __forceinline__ void group_scan32(int (&v)[N], Scan32Smem& sm, int (&tot)[N], int warp_in_group) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < N; ++c) v[c] = warp_incl_scan(v[c]);
  if (lane == 31) {
#pragma unroll
    for (int c = 0; c < N; ++c) sm.w[c][warp_in_group] = v[c];
  }
  G::sync();
#pragma unroll
  for (int c = 0; c < N; ++c) {
    const unsigned x = lane < G::kW ? (unsigned)sm.w[c][lane] : 0u;
    tot[c] = (int)__reduce_add_sync(kFull, x);
    v[c] += (int)__reduce_add_sync(kFull, lane < warp_in_group ? x : 0u);
  }
  G::sync();
}

}  // namespace rsd
