// pem.cuh -- CTA-cooperative PEM: the reference's analytic Alg. 1 cost
// (pkg/src/relsim/priority.py:163-218) without its item-by-item state machine.
//
// The reference scans items once, flushing a *segment* before item j when
// `utok_j + accum > cap or d_count + 1 > mns` and a *prefill sub-batch* when
// `utok_j > 0 and utok_j + p_utok > mnbt`, and sums one fp64 term per flushed
// batch in scan order.  Both flush rules are next-fit rules on prefix sums, so
// here:
//   1. one pass over the remainder builds inclusive prefix sums of utok (U),
//      remaining (REM) and the unprefilled count (UNP) with block scans
//      (coalesced loads, warp shuffles, one smem slot per warp);
//   2. every item i computes in parallel, by binary search on U, the item
//      that would close a segment / sub-batch opened at i (nseg[i], nsub[i]);
//   3. one thread follows the nseg chain (about size/mns hops), warps reduce
//      each segment's max remaining, and one thread follows the nsub chains,
//      adding the terms in exactly the reference's order with correctly
//      rounded fp64 operations (__dmul_rn/__dadd_rn; no FMA contraction).
// Every remainder item the engine produces has remaining >= 1 and prefilled
// items have utok 0 (remainder_items, priority.py:81-98); the unit entry point
// validates the same preconditions.
#pragma once
#include <stdint.h>

#include "block.cuh"

namespace rsd {

struct PemModel {
  double ap, bp, ad, bd;
  long long cap, mns, mnbt;
};

// Scratch for n items (generic pointers: shared or global memory).
struct PemBuf {
  long long* U;    // [n] inclusive prefix of utok
  long long* REM;  // [n] inclusive prefix of remaining
  int* UNP;        // [n] inclusive count of unprefilled items
  int* nsub;       // [n]
  int* nseg;       // [n]
  int* seg;        // [n+1] segment starts
  int* segmax;     // [n]
};

__host__ __device__ constexpr size_t pem_bytes_per_item() { return 8 + 8 + 4 + 4 + 4 + 4 + 4; }

__host__ __device__ inline PemBuf pem_carve(void* base, int cap_items) {
  char* p = (char*)base;
  PemBuf b;
  b.U = (long long*)p;
  p += sizeof(long long) * cap_items;
  b.REM = (long long*)p;
  p += sizeof(long long) * cap_items;
  b.UNP = (int*)p;
  p += sizeof(int) * cap_items;
  b.nsub = (int*)p;
  p += sizeof(int) * cap_items;
  b.nseg = (int*)p;
  p += sizeof(int) * cap_items;
  b.seg = (int*)p;
  p += sizeof(int) * (cap_items + 1);
  b.segmax = (int*)p;
  return b;
}

// rounded to 16 bytes so per-CTA slices of one allocation stay 8-byte aligned
__host__ __device__ inline size_t pem_buf_size(int cap_items) {
  return (pem_bytes_per_item() * (size_t)cap_items + 16 + 15) & ~(size_t)15;
}

struct PemShared {
  ScanSmem scan;
  double result;
  int n_items;
  int n_segs;
  int bad;
};

// smallest j in [lo, hi) with U[j] > x, else hi (U non-decreasing)
__device__ __forceinline__ int first_gt(const long long* U, int lo, int hi, long long x) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (U[mid] > x) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ double lin(double a, double x, double b) {
  return __dadd_rn(__dmul_rn(a, x), b);
}

// F::get(i, u, rem, pre) -> bool keep, for source index i in [0, n_src).
// Returns the PEM value (all threads), or NaN if an item has utok > cap.
template <class F>
__device__ double block_pem(const F& f, int n_src, const PemModel& m, PemBuf b, PemShared& sh) {
  const int tid = threadIdx.x;
  if (tid == 0) sh.bad = 0;
  long long cK = 0, cU = 0, cR = 0, cN = 0;
  for (int base = 0; base < n_src; base += kThreads) {
    const int i = base + tid;
    long long u = 0;
    int rem = 0, pre = 1;
    bool keep = false;
    if (i < n_src) keep = f.get(i, u, rem, pre);
    if (keep && u > m.cap) sh.bad = 1;
    long long v[4] = {keep ? 1LL : 0LL, keep ? u : 0LL, keep ? (long long)rem : 0LL,
                      (keep && !pre) ? 1LL : 0LL};
    long long tot[4];
    block_incl_scan<4>(v, sh.scan, tot);
    if (keep) {
      const int k = (int)(cK + v[0] - 1);
      b.U[k] = cU + v[1];
      b.REM[k] = cR + v[2];
      b.UNP[k] = (int)(cN + v[3]);
    }
    cK += tot[0];
    cU += tot[1];
    cR += tot[2];
    cN += tot[3];
  }
  const int n = (int)cK;
  __syncthreads();
  if (sh.bad) return __longlong_as_double(0x7FF8000000000000LL);
  if (n == 0) return 0.0;
  for (int i = tid; i < n; i += kThreads) {
    const long long before = i ? b.U[i - 1] : 0;
    const long long lim = (long long)i + m.mns < (long long)n ? (long long)i + m.mns : (long long)n;
    b.nseg[i] = first_gt(b.U, i + 1, (int)lim, before + m.cap);
    const long long thr = before + m.mnbt;
    // an item larger than mnbt on its own closes the batch at the next item with utok > 0
    b.nsub[i] = first_gt(b.U, i + 1, n, b.U[i] > thr ? b.U[i] : thr);
  }
  __syncthreads();
  if (tid == 0) {
    int s = 0, k = 0;
    while (s < n) {
      b.seg[k++] = s;
      s = b.nseg[s];
    }
    b.seg[k] = n;
    sh.n_segs = k;
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  const int nsegs = sh.n_segs;
  for (int k = warp; k < nsegs; k += kWarps) {
    const int s = b.seg[k], e = b.seg[k + 1];
    long long mx = 0;
    for (int j = s + lane; j < e; j += 32) {
      long long r = b.REM[j] - (j ? b.REM[j - 1] : 0);
      mx = r > mx ? r : mx;
    }
    mx = warp_max(mx);
    if (lane == 0) b.segmax[k] = (int)mx;
  }
  __syncthreads();
  if (tid == 0) {
    double total = 0.0;
    for (int k = 0; k < nsegs; ++k) {
      const int s = b.seg[k], e = b.seg[k + 1];
      int bb = s;
      for (;;) {
        const int nb = b.nsub[bb] < e ? b.nsub[bb] : e;
        const int unp = b.UNP[nb - 1] - (bb ? b.UNP[bb - 1] : 0);
        if (unp > 0) {
          const long long pu = b.U[nb - 1] - (bb ? b.U[bb - 1] : 0);
          total = __dadd_rn(total, lin(m.ap, (double)pu, m.bp));
        }
        bb = nb;
        if (bb >= e) break;
      }
      const long long rs = b.REM[e - 1] - (s ? b.REM[s - 1] : 0);
      const double t = __dadd_rn(__dmul_rn(m.ad, (double)rs), __dmul_rn(m.bd, (double)b.segmax[k]));
      total = __dadd_rn(total, t);
    }
    sh.result = total;
    sh.n_items = n;
  }
  __syncthreads();
  const double r = sh.result;
  __syncthreads();
  return r;
}

}  // namespace rsd
