// seg_pem.cuh -- PEM (priority.py:163-218) for a batch of remainders with the
// whole CTA: one block scan materialises the items, then one warp per
// *segment* finds the prefill sub-batch boundaries, and one thread per
// remainder adds the terms in the reference's order.
//
// Valid when no segment can be closed by the token capacity, i.e. when
// mns * max(utok) <= cap (checked on the host; otherwise warp_pem.cuh is
// used): segments are then closed only by the count rule
// `d_count + 1 > mns`, so remainder e's segment k is the fixed item range
// [k*mns - L_e, (k+1)*mns - L_e) after the L_e prefilled items summarised in
// PrefixSummary.  Inside a segment the sub-batch rule
// `utok_j > 0 and utok_j + p_utok > mnbt` is a next-fit chain on the prefix
// sums U, which a warp follows with 32-wide ballots over shared memory.
#pragma once
#include <stdint.h>

#include "block.cuh"
#include "pem.cuh"
#include "warp_pem.cuh"

namespace rsd {

struct SegBuf {
  long long* U;   // [NI] inclusive prefix of utok over the whole batch
  int* UNP;       // [NI] inclusive count of unprefilled items over the whole batch
  int* REM;       // [NI] remaining per item
  double* terms;  // [NI + J]
  int* jcnt;      // [J] terms written per job
  int* io;        // [nb+1] item offsets
  int* jo;        // [nb+1] job offsets
};

struct SegShared {
  ScanSmem scan;
};

// Item / job offsets of a batch (all threads; tid < nb supplies count(tid)).
template <class F>
__device__ void seg_offsets(const F& f, int nb, const PrefixSummary* ps, const PemModel& m, SegBuf b,
                            SegShared& sh) {
  const int tid = threadIdx.x;
  long long ni = 0, nj = 0;
  if (tid < nb) {
    ni = f.count(tid);
    const long long tot = ni + ps[tid].n;
    nj = tot > 0 ? (tot + m.mns - 1) / m.mns : 0;
  }
  long long v[2] = {ni, nj}, tot[2];
  block_incl_scan<2>(v, sh.scan, tot);
  if (tid < nb) {
    b.io[tid] = (int)(v[0] - ni);
    b.jo[tid] = (int)(v[1] - nj);
  }
  if (tid == 0) {
    b.io[nb] = (int)tot[0];
    b.jo[nb] = (int)tot[1];
  }
  __syncthreads();
}

// Materialise items: G(x, u, rem, pre) for item x of the concatenated batch;
// one inclusive scan of utok and of the unprefilled count over the batch.
template <class G>
__device__ void seg_materialize(const G& g, int NI, SegBuf b, SegShared& sh) {
  const int tid = threadIdx.x;
  long long carryU = 0, carryN = 0;
  for (int base = 0; base < NI; base += kThreads) {
    const int x = base + tid;
    long long u = 0;
    int rem = 0, pre = 1;
    if (x < NI) {
      g(x, u, rem, pre);
      b.REM[x] = rem;
    }
    long long v[2] = {u, (x < NI && !pre) ? 1LL : 0LL}, tot[2];
    block_incl_scan<2>(v, sh.scan, tot);
    if (x < NI) {
      b.U[x] = carryU + v[0];
      b.UNP[x] = (int)(carryN + v[1]);
    }
    carryU += tot[0];
    carryN += tot[1];
  }
  __syncthreads();
}

// Segment jobs (one warp each) and the ordered per-remainder sums.
template <class G>
__device__ void seg_jobs_and_sum(int nb, const PrefixSummary* ps, const PemModel& m, SegBuf b, const G& out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int J = b.jo[nb];
  for (int j = warp; j < J; j += kWarps) {
    int e = 0;
    while (b.jo[e + 1] <= j) ++e;
    const int k = j - b.jo[e];
    const int n = b.io[e + 1] - b.io[e];
    const int L = ps[e].n;
    const long long t0l = (long long)k * m.mns - L, t1l = (long long)(k + 1) * m.mns - L;
    const int t0 = t0l < 0 ? 0 : (int)t0l;
    const int t1 = t1l < n ? (int)t1l : n;
    // the batch scan runs across remainders: rebase on the item before t0
    const long long* U = b.U + b.io[e];
    const int* UNP = b.UNP + b.io[e];
    const int g0 = b.io[e] + t0;
    const long long Ub = g0 > 0 ? b.U[g0 - 1] : 0, Nb = g0 > 0 ? b.UNP[g0 - 1] : 0;
    double* out_terms = b.terms + b.io[e] + b.jo[e] + k + t0;
    int nterm = 0;
    int bb = t0;
    while (bb < t1) {
      // sub-batch [bb, nbk): closes before the first later item j with
      // utok_j > 0 and utok(bb..j) > mnbt (priority.py:205-208)
      const long long before = bb > t0 ? U[bb - 1] - Ub : 0;
      const long long ub = U[bb] - Ub;
      const long long thr = ub - before > m.mnbt ? ub : before + m.mnbt;
      int nbk = t1;
      for (int base = bb + 1; base < t1; base += 32) {
        const int x = base + lane;
        const bool hit = x < t1 && U[x] - Ub > thr;
        const unsigned msk = __ballot_sync(kFull, hit);
        if (msk) {
          nbk = base + __ffs(msk) - 1;
          break;
        }
      }
      const long long unp = (UNP[nbk - 1] - Nb) - (bb > t0 ? UNP[bb - 1] - Nb : 0);  // any unprefilled item
      if (unp > 0 && lane == 0) {
        const long long pu = (U[nbk - 1] - Ub) - before;
        out_terms[nterm] = lin(m.ap, (double)pu, m.bp);
      }
      nterm += unp > 0;
      bb = nbk;
    }
    // decode term: sum and max of remaining over the segment
    long long rs = 0, mx = 0;
    for (int x = t0 + lane; x < t1; x += 32) {
      const long long r = b.REM[b.io[e] + x];
      rs += r;
      mx = r > mx ? r : mx;
    }
    rs = warp_sum(rs);
    mx = warp_max(mx);
    if (k == 0) {
      rs += ps[e].rsum;
      mx = ps[e].rmax > mx ? ps[e].rmax : mx;
    }
    if (lane == 0) {
      out_terms[nterm] = __dadd_rn(__dmul_rn(m.ad, (double)rs), __dmul_rn(m.bd, (double)mx));
      b.jcnt[j] = nterm + 1;
    }
  }
  __syncthreads();
  // ordered sums: segment by segment, terms in emission order
  if (tid < nb) {
    double total = 0.0;
    const int nj = b.jo[tid + 1] - b.jo[tid];
    for (int k = 0; k < nj; ++k) {
      const long long t0l = (long long)k * m.mns - ps[tid].n;
      const int t0 = t0l < 0 ? 0 : (int)t0l;
      const double* tt = b.terms + b.io[tid] + b.jo[tid] + k + t0;
      const int cnt = b.jcnt[b.jo[tid] + k];
      int i = 0;
      for (; i + 4 <= cnt; i += 4) {  // independent loads, dependent adds
        const double x0 = tt[i], x1 = tt[i + 1], x2 = tt[i + 2], x3 = tt[i + 3];
        total = __dadd_rn(total, x0);
        total = __dadd_rn(total, x1);
        total = __dadd_rn(total, x2);
        total = __dadd_rn(total, x3);
      }
      for (; i < cnt; ++i) total = __dadd_rn(total, tt[i]);
    }
    out(tid, total);
  }
  __syncthreads();
}

// F::count(e), F::item(e, i, u, rem, pre); the whole pipeline for one batch.
template <class F, class G>
__device__ void seg_pem_batch(const F& f, int nb, const PrefixSummary* ps, const PemModel& m, SegBuf b,
                              SegShared& sh, const G& out) {
  seg_offsets(f, nb, ps, m, b, sh);
  const int NI = b.io[nb];
  struct ByItem {
    const F& f;
    const int* io;
    int nb;
    __device__ void operator()(int x, long long& u, int& rem, int& pre) const {
      int e = 0;
      while (io[e + 1] <= x) ++e;
      f.item(e, x - io[e], u, rem, pre);
    }
  };
  seg_materialize(ByItem{f, b.io, nb}, NI, b, sh);
  seg_jobs_and_sum(nb, ps, m, b, out);
}

}  // namespace rsd
