// dpu.cuh -- the Dynamic Priority Updater (priority.py:238-339) for one
// scheduler iteration, run by the whole CTA.
//
// Only relQueries the reference would re-estimate are touched: its reuse rule
// (priority.py:261-266) keeps the previous value for every live relQuery that
// was live last time and has no prefilled or finished row, so the estimated
// set is the partially prefilled live relQueries (the sorted act list) plus
// this iteration's arrivals, in admission order -- the order the numpy RNG
// stream is consumed in.  Per batch of up to kEstBatch relQueries:
//   1. metadata + draw offsets (block scan);
//   2. sample_cache_miss_ratio's Generator.choice draws for the whole batch
//      in parallel from PCG64 jump-ahead, with a sequential replay if any
//      Lemire rejection occurred;
//   3. ratios (Floyd's set per relQuery; utok of an unprefilled row is
//      tok - B*m exactly, prefix_cache.py:70-93);
//   4. PEM: running rows enter as a prefilled summary, unprefilled rows as
//      utok_approx items; segment-parallel (seg_pem.cuh) when segments can
//      only close by count, else one warp per relQuery (warp_pem.cuh).
// Then the starvation override for wholly-waiting relQueries.
#pragma once
#include "engine_state.cuh"

namespace rsd {

// Unprefilled rows [q, size) of a relQuery as PEM items (remainder_items,
// priority.py:81-98): utok_approx = min(tok, floor(tok*ratio + 0.5))
// (prefix_cache.py:172-176), remaining = output_limit, not prefilled.
__device__ __forceinline__ long long utok_approx(long long tk, double ratio) {
  const long long a = (long long)floor(__dadd_rn(__dmul_rn((double)tk, ratio), 0.5));
  return tk < a ? tk : a;
}

struct UnprefItems {
  const int* tok;
  int base, ol;
  double ratio;
  __device__ __forceinline__ void item(int t, long long& u, int& rem, int& pre) const {
    u = utok_approx(tok[base + t], ratio);
    rem = ol;
    pre = 0;
  }
};

struct EstItems {
  const int* tok;
  const int* off;
  const int* q;
  const int* nunp;
  const int* ol;
  const double* ratio;
  __device__ __forceinline__ int count(int e) const { return nunp[e]; }
  __device__ __forceinline__ void item(int e, int i, long long& u, int& rem, int& pre) const {
    u = utok_approx(tok[off[e] + q[e] + i], ratio[e]);
    rem = ol[e];
    pre = 0;
  }
};

struct PrioOut {
  double* prio;
  const int* rank;
  __device__ __forceinline__ void operator()(int e, double v) const { prio[rank[e]] = v; }
};

// Sequential sample_cache_miss_ratio (prefix_cache.py:141-169) for relQuery a
// (thread 0; the fallback after a Lemire rejection).
__device__ double sample_ratio_seq(Pcg64& g, const TraceDev& T, const RqView& rq, const Params& P, int a,
                                   uint32_t* idx) {
  const int off = rq.off[a];
  const int size = rq.off[a + 1] - off;
  const int q = rq.q[a];
  const int n = size - q;  // unprefilled rows = [q, size) (SURVEY A-inv1)
  if (n <= 0) return 0.0;
  const long long mh = P.cfg.block_size * (long long)rq.m[a];
  const int k = (int)(P.cfg.sample_size < n ? P.cfg.sample_size : n);
  long long usum = 0, tsum = 0;
  if (k < n) {  // idx: shared scratch (a local array would give the kernel a stack frame)
    choice_floyd(g, (uint32_t)n, (uint32_t)k, idx);
    for (int i = 0; i < k; ++i) {
      const long long t = T.tok[off + q + (int)idx[i]];
      usum += t - mh;
      tsum += t;
    }
  } else {
    for (int i = 0; i < n; ++i) {
      const long long t = T.tok[off + q + i];
      usum += t - mh;
      tsum += t;
    }
  }
  return __ddiv_rn((double)usum, (double)tsum);
}


// Cold path: sequential numpy replay for relQueries [0, n_est) of this
// iteration's estimated list (after a Lemire rejection).
__device__ void ratios_sequential(const Params& P, const TraceDev& T, Shared& S, int e0, int n_est, int n_act) {
  Ctl& c = S.c;
  Pcg64 g = Pcg64::from(c.rng);
  for (int e = 0; e < n_est; ++e) {
    const int ge = e0 + e;
    const int ae = ge < n_act ? c.act[ge] : S.new_lo + (ge - n_act);
    S.est_ratio[e] = sample_ratio_seq(g, T, S.rq, P, ae, S.floyd_idx);
  }
  c.rng = g.to();
}

// sample_cache_miss_ratio's sampled rows (prefix_cache.py:157-164): Floyd's
// set from the K bounded draws of one choice(n, K) call -- a draw equal to an
// earlier member is replaced by n-K+d; the Fisher-Yates draws after them only
// permute the set -- and the sum of the sampled rows' tok.
template <int K>
__device__ __forceinline__ long long floyd_tok_sum(const int* tok, const unsigned* draws, uint32_t n) {
  uint32_t idx[K];
#pragma unroll
  for (int d = 0; d < K; ++d) {
    const uint32_t v = draws[d];
    bool found = false;
#pragma unroll
    for (int x = 0; x < d; ++x) found |= idx[x] == v;
    idx[d] = found ? n - K + d : v;
  }
  int t[K];
#pragma unroll
  for (int d = 0; d < K; ++d) t[d] = tok[idx[d]];
  long long sum = 0;
#pragma unroll
  for (int d = 0; d < K; ++d) sum += t[d];
  return sum;
}

__device__ __noinline__ long long floyd_tok_sum_any(const int* tok, const unsigned* draws, uint32_t n, int K) {
  uint32_t idx[kMaxSample];
  long long sum = 0;
  for (int d = 0; d < K; ++d) {
    const uint32_t v = draws[d];
    bool found = false;
    for (int x = 0; x < d; ++x) found |= idx[x] == v;
    idx[d] = found ? n - (uint32_t)K + (uint32_t)d : v;
    sum += tok[idx[d]];
  }
  return sum;
}

// Fast path for the common steady state (few re-estimated relQueries, PEM
// segments closed by count only, mns <= 256, sample size <= 16): two block
// barriers in total.
//   * every warp derives the per-relQuery metadata and the draw / segment
//     offsets itself (lane e = relQuery e, warp scans; no barrier);
//   * warp 0 replays the numpy draws from jump-ahead (lane per position) and
//     computes the sample ratios; the other warps build the running-row
//     summaries;
//   * one warp per PEM segment materialises its utok prefix, follows the
//     sub-batch chain with ballots, and emits its terms;
//   * lane e of warp 0 adds relQuery e's terms in the reference's order.
// Returns false (nothing changed) when the preconditions do not hold.
// Processes the estimated relQueries [e0, e0 + n) of this iteration's list
// (act then arrivals) for the largest n <= min(32, e1 - e0) whose PEM
// segments fit kMaxJobs; returns n (0 if even one does not fit).
template <bool kC>
__device__ int dpu_small(const Params& P, const TraceDev& T, Shared& S, const PemModel& pm, int e0, int e1) {
  Ctl& c = S.c;
  const RqView rq = S.rq;  // by value: the table pointers stay in registers across the barriers
  const rs_config& cfg = P.cfg;
  const int tid = threadIdx.x, lane = tid & 31, warp = opaque_warp();
  const int n_act = c.n_act;
  int n_est = e1 - e0 < kSmallEst ? e1 - e0 : kSmallEst;
  const int Ssz = kC ? 8 : (int)cfg.sample_size;  // kC: the default sample size (engine.py:150)
  const int dper = 2 * Ssz - 1;
  // per-warp metadata: lane e holds relQuery e0 + e
  int a = 0, base = 0, nunp = 0, ol = 0, mcb = 0, L = 0, dcnt = 0, nj = 0;
  bool own = false;  // sharded pool: only the owner estimates (shard.cuh); the RNG positions count every one
  if (lane < n_est) {
    const int ge = e0 + lane;
    a = ge < n_act ? c.act[ge] : S.new_lo + (ge - n_act);
    own = kC || T.shard_world == 1 || a % T.shard_world == T.shard_rank;
    const int off = rq.off[a];
    const int q = rq.q[a];
    base = off + q;
    nunp = rq.off[a + 1] - base;
    ol = rq.ol[a];
    mcb = rq.m[a];
    L = rq.nrun[a];  // running rows = the live prefilled rows (prefilled summary)
    dcnt = nunp > Ssz ? dper : 0;  // choice() only when k = S < n (prefix_cache.py:157-158)
    const unsigned tot = (unsigned)(nunp + L);  // segments = ceil(tot / mns) by multiply-shift (exact: tot < 2^32/mns)
    nj = tot > 0 && own ? (int)(((unsigned long long)(tot + (unsigned)pm.mns - 1u) * P.mns_magic) >> 32) : 0;
  }
  // draw and PEM-segment offsets in one warp scan: (dcnt << 16) | nj (per-warp
  // totals stay below 2^16: dcnt <= 2*16-1 and nj <= kMaxJobs per kept relQuery)
  int incl = warp_incl_scan((dcnt << 16) | nj);
  {  // keep the prefix of relQueries whose segments fit the job buffers
    const int fit = __popc(__ballot_sync(kFull, lane < n_est && (incl & 0xFFFF) <= kMaxJobs));
    if (fit < n_est) {
      n_est = fit;
      if (lane >= n_est) dcnt = nj = nunp = 0;
      incl = warp_incl_scan((dcnt << 16) | nj);
    }
  }
  if (n_est == 0) return 0;
  const int jincl = incl & 0xFFFF, dincl = incl >> 16;
  const int doff = dincl - dcnt, jo = jincl - nj;
  const int tot_incl = __shfl_sync(kFull, incl, 31);
  const int D = tot_incl >> 16, J = tot_incl & 0xFFFF;
  if (warp == 0) {  // PEM items' tok + sampled tok
    const unsigned nb = own ? (unsigned)(nunp + (nunp > Ssz ? Ssz : nunp)) : 0u;
    const unsigned tot_b = __reduce_add_sync(kFull, nb);
    if (lane == 0) c.alg_bytes += 4LL * tot_b;
  }
  phase_mark(c, 5);
  if (warp == 0) {
    // numpy next32 stream positions [0, D) -> bounded draws
    const unsigned h0 = c.rng.has_uint32;
    const U128 s0{c.rng.state_hi, c.rng.state_lo};
    bool rej = false;
    {  // owner lookup tables: the k-th relQuery that draws owns positions [k*dper, (k+1)*dper)
      const unsigned dm = __ballot_sync(kFull, lane < n_est && dcnt > 0);
      if (lane < n_est) {
        S.est_doff[lane] = dcnt > 0 ? doff : 0x7FFFFFFF;
        S.est_nunp[lane] = nunp;
        if (dcnt > 0) S.est_drawer[__popc(dm & ((1u << lane) - 1u))] = lane;
      }
    }
    __syncwarp();
    // lane l owns 64-bit output l of each 32-output round: state_{32r+l+1} =
    // A^(l+1) state_{32r} + C_(l+1) (one 128-bit multiply-add from the
    // consecutive-step table), whose low / high halves are next32 values
    // 2l and 2l+1 after the buffered one
    const int cnt32 = D - (int)h0 > 0 ? D - (int)h0 : 0;  // fresh next32 values
    const int n64 = (cnt32 + 1) >> 1;
    U128 sb = s0;
    U128 s_end = s0;
    uint64_t out_end = 0;
    __syncwarp();
    phase_mark(c, 16);
    for (int r0 = 0; r0 < n64; r0 += 32) {
      const U128 st = add128(mul128(S.jstep[lane].a, sb), S.jstep[lane].c);
      const uint64_t out = pcg_output(st);
      __syncwarp();
      phase_mark(c, 17);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int p = (int)h0 + 2 * (r0 + lane) + half;
        if (p < D) {
          const uint32_t v = half ? (uint32_t)(out >> 32) : (uint32_t)out;
          const int kq = (int)(((unsigned)p * P.dper_magic) >> 16);  // p / dper (exact: p < 2^16 / dper)
          const int d = p - kq * dper;
          const uint32_t ne = (uint32_t)S.est_nunp[S.est_drawer[kq]];
          const uint32_t bound = d < Ssz ? ne - (uint32_t)Ssz + (uint32_t)d : (uint32_t)(Ssz - 1 - (d - Ssz));
          const uint32_t excl = bound + 1u;
          const uint64_t mm = (uint64_t)v * excl;
          const uint32_t left = (uint32_t)mm;
          if (left < excl) {  // rare: only then can Lemire reject
            if (left < (0xFFFFFFFFu - bound) % excl) rej = true;
          }
          S.small.draws[p] = (uint32_t)(mm >> 32);
        }
      }
      __syncwarp();
      phase_mark(c, 18);
      const int last = n64 - 1 - r0;  // lane holding the final state, if in this round
      if (last < 32) {
        s_end.hi = __shfl_sync(kFull, st.hi, last);
        s_end.lo = __shfl_sync(kFull, st.lo, last);
        out_end = __shfl_sync(kFull, out, last);
      }
      sb.hi = __shfl_sync(kFull, st.hi, 31);
      sb.lo = __shfl_sync(kFull, st.lo, 31);
    }
    if (h0 && D > 0 && lane == 0) {  // position 0 is the buffered half-word
      const uint32_t v = c.rng.uinteger;
      int e = 0;
      for (int x = 0; x < n_est; ++x)
        if (S.est_doff[x] <= 0) e = x;
      const uint32_t ne = (uint32_t)S.est_nunp[e];
      const uint32_t bound = ne - (uint32_t)Ssz;  // d = 0: Floyd's first bound n - k
      const uint32_t excl = bound + 1u;
      const uint64_t mm = (uint64_t)v * excl;
      const uint32_t left = (uint32_t)mm;
      if (left < excl && left < (0xFFFFFFFFu - bound) % excl) rej = true;
      S.small.draws[0] = (uint32_t)(mm >> 32);
    }
    rej = __any_sync(kFull, rej);
    __syncwarp();
    phase_mark(c, 6);
    if (rej) {  // replay sequentially: a rejection shifts every later draw
      if (lane == 0) ratios_sequential(P, T, S, e0, n_est, n_act);
    } else {
      if (lane < n_est && own) {  // sample_cache_miss_ratio (prefix_cache.py:141-169)
        const long long mh = (kC ? 16 : cfg.block_size) * (long long)mcb;  // exact utok = tok - B*m
        double ratio = 0.0;
        if (nunp > 0) {
          long long usum = 0, tsum = 0;
          if (nunp <= Ssz) {
            for (int i = 0; i < nunp; ++i) {
              const long long t = T.tok[base + i];
              usum += t - mh;
              tsum += t;
            }
          } else if (Ssz == 8) {  // the default sample size: Floyd's set in registers
            tsum = floyd_tok_sum<8>(T.tok + base, S.small.draws + doff, (uint32_t)nunp);
            usum = tsum - 8 * mh;
          } else {  // other sizes: rolled (the hot path keeps one specialised copy)
            tsum = floyd_tok_sum_any(T.tok + base, S.small.draws + doff, (uint32_t)nunp, Ssz);
            usum = tsum - (long long)Ssz * mh;
          }
          ratio = __ddiv_rn((double)usum, (double)tsum);
        }
        S.est_ratio[lane] = ratio;
      }
      __syncwarp();
      phase_mark(c, 15);
      if (lane == 0 && D > 0) {  // advance the generator past the D values
        // numpy's next32 buffer: the high half of the last 64-bit output stays in
        // `uinteger` whether or not it was consumed (an even count leaves it stale)
        if (cnt32 == 0) {
          c.rng.has_uint32 = 0;
        } else {
          c.rng.state_hi = s_end.hi;
          c.rng.state_lo = s_end.lo;
          c.rng.has_uint32 = cnt32 & 1;
          c.rng.uinteger = (uint32_t)(out_end >> 32);
        }
      }
    }
  } else {
    // running-row summaries (count, sum and max of remaining) for relQueries with running rows
    for (int e = warp - 1; e < n_est; e += kWarps - 1) {
      const int ae = __shfl_sync(kFull, a, e);
      const int Le = __shfl_sync(kFull, L, e);
      const int ole = __shfl_sync(kFull, ol, e);
      const bool owne = __shfl_sync(kFull, (int)own, e);
      PrefixSummary ps{0, 0, 0};
      if (Le > 0 && owne) {
        long long rs = 0, mx = 0;
#pragma unroll 1
        for (int j = lane; j < c.n_run; j += 32)
          if (c.run_rank[j] == ae) {
            const long long r = ole - c.run_gen[j];
            rs += r;
            mx = r > mx ? r : mx;
          }
        ps.n = Le;  // sums of at most mns rows of remaining <= output_limit: 32-bit hardware reductions
        ps.rsum = __reduce_add_sync(kFull, (unsigned)rs);
        ps.rmax = (int)__reduce_max_sync(kFull, (unsigned)mx);
      }
      if (lane == 0) S.est_ps[e] = ps;
    }
  }
  // one PEM segment per warp 1..15 (warp 0 is busy with the RNG above); the
  // first segment's tok loads are issued before the barrier, under the RNG
  // replay.  One loop with the barrier in its first pass keeps a single copy
  // of the job setup in the instruction stream.
  static_assert(kSmallMns <= 8 * 32, "items per lane");
  for (int j = warp - 1, first = 1;; j += kWarps - 1, first = 0) {
    const bool act = warp > 0 && j < J;
    int e = 0, k = 0, ne = 0, Le = 0, basee = 0, ole = 0, t0 = 0, nloc = 0;
    int uv[8];
    if (act) {
      // the job's relQuery: the last one (lane) whose segments start at or before j
      const unsigned em = __ballot_sync(kFull, lane < n_est && jo <= j && nj > 0);
      e = 31 - __clz(em);
      k = j - __shfl_sync(kFull, jo, e);
      ne = __shfl_sync(kFull, nunp, e);
      Le = __shfl_sync(kFull, L, e);
      basee = __shfl_sync(kFull, base, e);
      ole = __shfl_sync(kFull, ol, e);
      const int mns = (int)pm.mns;
      t0 = k * mns - Le < 0 ? 0 : k * mns - Le;
      nloc = ((k + 1) * mns - Le < ne ? (k + 1) * mns - Le : ne) - t0;
    }
    // utok prefix of the segment: lane l owns items [l*per, l*per + per), per <= 8 (nloc <= mns)
    const int per = (nloc + 31) >> 5, x0 = lane * per;
#pragma unroll
    for (int i = 0; i < 8; ++i) uv[i] = (act && i < per && x0 + i < nloc) ? T.tok[basee + t0 + x0 + i] : 0;
    if (first) {
      __syncthreads();
      phase_mark(c, 7);
    }
    if (!act) break;
    const double ratio = S.est_ratio[e];
    int* Uw = S.small.U[warp];
    {
      int ls = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uv[i] = uv[i] ? (int)utok_approx(uv[i], ratio) : 0;
        ls += uv[i];
      }
      int run = warp_incl_scan(ls) - ls;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        run += uv[i];
        if (i < per && x0 + i < nloc) Uw[x0 + i] = run;
      }
    }
    __syncwarp();
    double* tj = S.small.terms + j * kJobTerms;
    double* spill = T.term_spill + (size_t)j * (kSmallMns + 1);
    int nterm = 0;
    int bb = 0;
    int my_end = 0;  // lane l < 32: one past the last row of sub-batch l (its term is computed after the chain)
    while (bb < nloc) {
      // every item is unprefilled, so every sub-batch is non-empty: one p-term each
      const int before = bb ? Uw[bb - 1] : 0;
      const int ub = Uw[bb];
      const int thr = ub - before > pm.mnbt ? ub : before + (int)pm.mnbt;
      int nb = nloc;
      for (int b2 = bb + 1; b2 < nloc; b2 += 64) {  // 64 candidates per round: a sub-batch is ~40-60 rows
        const int x = b2 + lane, y = x + 32;
        const bool hx = x < nloc && Uw[x] > thr, hy = y < nloc && Uw[y] > thr;
        const unsigned mx = __ballot_sync(kFull, hx), my = __ballot_sync(kFull, hy);
        if (mx | my) {
          nb = mx ? b2 + __ffs(mx) - 1 : b2 + 32 + __ffs(my) - 1;
          break;
        }
      }
      if (nterm < 32) {
        if (lane == nterm) my_end = nb;
      } else if (lane == 0) {  // rare: more than 32 sub-batches in one segment
        const double t = lin(pm.ap, (double)(Uw[nb - 1] - before), pm.bp);
        if (nterm < kJobTerms) tj[nterm] = t;
        else spill[nterm] = t;
      }
      ++nterm;
      bb = nb;
    }
    {  // the p-terms of the first 32 sub-batches, one lane each, off the chain's critical path
      static_assert(kJobTerms >= 32, "terms 0..31 live in shared memory");
      const int beg = __shfl_up_sync(kFull, my_end, 1);
      if (lane < nterm && lane < 32) {
        const int b0 = lane ? beg : 0;
        tj[lane] = lin(pm.ap, (double)(Uw[my_end - 1] - (b0 ? Uw[b0 - 1] : 0)), pm.bp);
      }
    }
    if (lane == 0) {
      long long rs = (long long)nloc * ole;
      long long mx = nloc > 0 ? ole : 0;
      if (k == 0) {
        rs += S.est_ps[e].rsum;
        mx = S.est_ps[e].rmax > mx ? S.est_ps[e].rmax : mx;
      }
      const double t = __dadd_rn(__dmul_rn(pm.ad, (double)rs), __dmul_rn(pm.bd, (double)mx));
      if (nterm < kJobTerms) tj[nterm] = t;
      else spill[nterm] = t;
      S.small.nterm[j] = nterm + 1;
    }
    __syncwarp();
  }
  __syncthreads();
  phase_mark(c, 8);
  if (warp == 0 && lane < n_est && own) {  // ordered sums, relQuery by relQuery
    double total = 0.0;
    for (int j = jo; j < jo + nj; ++j) {
      const int cnt = S.small.nterm[j];
      const double* tj = S.small.terms + j * kJobTerms;
      const double* spill = T.term_spill + (size_t)j * (kSmallMns + 1);
      const int nsm = cnt < kJobTerms ? cnt : kJobTerms;
#pragma unroll 4
      for (int i = 0; i < nsm; ++i) total = __dadd_rn(total, tj[i]);
#pragma unroll 1
      for (int i = nsm; i < cnt; ++i) total = __dadd_rn(total, spill[i]);  // segments of > 31 sub-batches
    }
    rq.prio[a] = total;
  }
  // (the caller's barrier orders these writes before the waiting order)
  return n_est;
}

// Pipelined priority update (engine_kernel<true, true>, warps kMWarps..15 =
// group D).  While group M executes this iteration's decided action, group D
// computes the NEXT iteration's re-estimates of the partially prefilled
// relQueries (the c.act list, priority.py:261-303) from the state that action
// leaves -- known before it is applied:
//   prefill of rows [q, q+n) of the head h: q_h += n, h's chain becomes fully
//     resident (m_h = chain_h: every insert of the batch pins it), the n rows
//     join the running set with remaining = output_limit, and h joins the list
//     if this is its first prefill (engine.py:315-341);
//   decode: every running row's remaining drops by one and finished rows leave
//     (engine.py:343-363); a relQuery with no unprefilled and no running row
//     left retires and is not updated;
//   idle: nothing changes.
// The sampled ratios use the chain lengths seen now; the prefill advance may
// evict another relQuery's chain (cache_model.cuh), so spec_commit checks every
// chain length used against the advance's result.  The numpy draws continue
// from this iteration's final generator state, in the same list order.  Every
// input is read before the handoff barrier (group M writes none of them
// earlier); results go to S.spec_* and are committed after the join.  Only the
// fast path's shape (<= kSmallEst relQueries, <= kMaxJobs PEM segments, no
// Lemire rejection) is speculated; otherwise the next iteration runs
// dpu_update in place.
template <bool kPart>
__device__ void dpu_spec(const Params& P, const TraceDev& T, Shared& S, const int action, const int h, const int nh,
                         const bool allowed) {
  Ctl& c = S.c;
  const RqView rq = S.rq;
  const int lane = threadIdx.x & 31, gw = opaque_warp() - kMWarps;
  const bool pf = action == RS_ACTION_PREFILL, dec = action == RS_ACTION_DECODE;
  dphase_mark(c, -1);
  const int n_act = c.n_act;
  const bool join = pf && rq.q[h] == 0;  // h's first prefill: it joins the list
  // kPart, more than kSmallEst entries: the first kSmallEst are computed here and
  // the next iteration's phase B estimates the rest in place, continuing the
  // generator (else such an update runs wholly in place)
  const int n_full = n_act + (join ? 1 : 0);
  const int n_est = kPart && n_full > kSmallEst ? kSmallEst : n_full;
#ifdef RS_NO_SPEC  // experiment: the pipelined update disabled (every update runs in place)
  const bool no_spec = true;
#else
  const bool no_spec = false;
#endif
  if (no_spec || !allowed || n_est > kSmallEst || n_est == 0) {  // group-uniform
    if (threadIdx.x == kMWarps * 32) {
      S.spec_valid = !no_spec && n_est == 0 && allowed;  // nothing to re-estimate: trivially done
      S.spec_n = 0;
      if constexpr (kPart) S.spec_part = 0;
      S.spec_rng = c.rng;
      S.spec_alg = 0;
    }
    handoff_arrive();
    return;
  }
  constexpr int Ssz = 8, dper = 2 * Ssz - 1;  // kC: the default sample size (engine.py:150)
  PemModel pm;
  pm.ap = P.pol.alpha_p;
  pm.bp = P.pol.beta_p;
  pm.ad = P.pol.alpha_d;
  pm.bd = P.pol.beta_d;
  pm.cap = P.cfg.cap;
  pm.mns = P.cfg.max_num_seqs;
  pm.mnbt = P.cfg.max_num_batched_tokens;
  // 0. the list (act, with h inserted in rank order on its first prefill) and
  //    each entry's state after the advance; the draw offsets (they depend on
  //    the unprefilled counts only)
  if (gw == 0) {
    const int x = lane < n_act ? c.act[lane] : 0x7FFFFFFF;
    const int pos = join ? __popc(__ballot_sync(kFull, x < h)) : 32;
    const int xm1 = __shfl_up_sync(kFull, x, 1);
    const int a = lane < pos ? x : (lane == pos ? h : xm1);
    int nunp = 0;
    if (lane < n_est) {
      const int off = rq.off[a], size = rq.off[a + 1] - off;
      const bool isH = pf && a == h;
      const int q = rq.q[a] + (isH ? nh : 0);
      const int ol = rq.ol[a];
      nunp = size - q;
      S.spec_rank[lane] = a;
      S.spec_m[lane] = isH ? rq.chain[a] : rq.m[a];
      S.spec_nunp[lane] = nunp;
      S.spec_base[lane] = off + q;
      S.spec_ol[lane] = ol;
      S.spec_L[lane] = isH ? nh : 0;  // the batch's rows join the running set, remaining = output_limit
      S.spec_rsum[lane] = isH ? nh * ol : 0;
      S.spec_rmax[lane] = isH ? ol : 0;
    }
    const int dcnt = lane < n_est && nunp > Ssz ? dper : 0;  // choice() only when k = S < n
    const int dincl = warp_incl_scan(dcnt);
    const unsigned dm = __ballot_sync(kFull, dcnt > 0);
    if (lane < n_est) {
      S.est_doff[lane] = dcnt > 0 ? dincl - dcnt : 0x7FFFFFFF;
      S.est_nunp[lane] = nunp;
      if (dcnt > 0) S.est_drawer[__popc(dm & ((1u << lane) - 1u))] = lane;
    }
    if (lane == 31) S.spec_draws = dincl;
    {  // the PEM items' and the sampled rows' tok
      const unsigned nb = (unsigned)(nunp + (nunp > Ssz ? Ssz : nunp));
      const unsigned tot_b = __reduce_add_sync(kFull, nb);
      if (lane == 0) S.spec_alg = 4LL * tot_b;
    }
    if (lane == 0) {
      S.spec_n = n_est;
      if constexpr (kPart) S.spec_part = n_full > n_est;
      S.spec_valid = 1;
    }
  }
  GD::sync();
  dphase_mark(c, 5);
  if (gw == 0) {
    handoff_arrive();  // warp 0 reads no state group M changes from here on
    // 1a. the numpy draws (positions [0, D) of next32, from the generator after this
    //     iteration's update) and the sampled ratios, while warps 1.. build the summaries
    const int D = S.spec_draws;
    const rs_pcg64_state r0 = c.rng;
    const unsigned h0 = r0.has_uint32;
    const U128 s0{r0.state_hi, r0.state_lo};
    bool rej = false;
    const int cnt32 = D - (int)h0 > 0 ? D - (int)h0 : 0;
    const int n64 = (cnt32 + 1) >> 1;
    U128 sb = s0, s_end = s0;
    uint64_t out_end = 0;
    for (int r0i = 0; r0i < n64; r0i += 32) {
      const U128 st = add128(mul128(S.jstep[lane].a, sb), S.jstep[lane].c);
      const uint64_t out = pcg_output(st);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int p = (int)h0 + 2 * (r0i + lane) + half;
        if (p < D) {
          const uint32_t v = half ? (uint32_t)(out >> 32) : (uint32_t)out;
          const int kq = (int)(((unsigned)p * P.dper_magic) >> 16);  // p / dper
          const int d = p - kq * dper;
          const uint32_t ne = (uint32_t)S.est_nunp[S.est_drawer[kq]];
          const uint32_t bound = d < Ssz ? ne - (uint32_t)Ssz + (uint32_t)d : (uint32_t)(Ssz - 1 - (d - Ssz));
          const uint32_t excl = bound + 1u;
          const uint64_t mm = (uint64_t)v * excl;
          const uint32_t left = (uint32_t)mm;
          if (left < excl && left < (0xFFFFFFFFu - bound) % excl) rej = true;
          S.small.draws[p] = (uint32_t)(mm >> 32);
        }
      }
      const int last = n64 - 1 - r0i;
      if (last < 32) {
        s_end.hi = __shfl_sync(kFull, st.hi, last);
        s_end.lo = __shfl_sync(kFull, st.lo, last);
        out_end = __shfl_sync(kFull, out, last);
      }
      sb.hi = __shfl_sync(kFull, st.hi, 31);
      sb.lo = __shfl_sync(kFull, st.lo, 31);
    }
    if (h0 && D > 0 && lane == 0) {  // position 0 is the buffered half-word
      const uint32_t bound = (uint32_t)S.est_nunp[S.est_drawer[0]] - (uint32_t)Ssz;
      const uint32_t excl = bound + 1u;
      const uint64_t mm = (uint64_t)r0.uinteger * excl;
      const uint32_t left = (uint32_t)mm;
      if (left < excl && left < (0xFFFFFFFFu - bound) % excl) rej = true;
      S.small.draws[0] = (uint32_t)(mm >> 32);
    }
    rej = __any_sync(kFull, rej);
    __syncwarp();
    dphase_mark(c, 9);
    if (rej) {  // a rejection shifts every later draw: the next iteration replays it in place
      if (lane == 0) S.spec_valid = 0;
    } else {
      if (lane < n_est) {  // sample_cache_miss_ratio (prefix_cache.py:141-169), utok = tok - B*m
        const int nunp = S.spec_nunp[lane], base = S.spec_base[lane];
        const long long mh = 16LL * S.spec_m[lane];
        double ratio = 0.0;
        if (nunp > 0) {
          long long usum = 0, tsum = 0;
          if (nunp <= Ssz) {
            for (int i = 0; i < nunp; ++i) {
              const long long t = T.tok[base + i];
              usum += t - mh;
              tsum += t;
            }
          } else {
            tsum = floyd_tok_sum<8>(T.tok + base, S.small.draws + S.est_doff[lane], (uint32_t)nunp);
            usum = tsum - 8 * mh;
          }
          ratio = __ddiv_rn((double)usum, (double)tsum);
        }
        S.est_ratio[lane] = ratio;
      }
      dphase_mark(c, 11);
      if (lane == 0) {
        rs_pcg64_state r = r0;
        if (D > 0) {  // numpy's half-word buffer (see dpu_small)
          if (cnt32 == 0) {
            r.has_uint32 = 0;
          } else {
            r.state_hi = s_end.hi;
            r.state_lo = s_end.lo;
            r.has_uint32 = cnt32 & 1;
            r.uinteger = (uint32_t)(out_end >> 32);
          }
        }
        S.spec_rng = r;
      }
    }
  } else {
    // 1b. running-row summaries after the advance (decode: gen + 1, finished rows leave)
    //     two rows per thread in one pass (224 threads, up to 448 rows): their loads and
    //     searches overlap instead of a second round
    constexpr int kSum = (kDWarps - 1) * 32;
    const int t = threadIdx.x - (kMWarps + 1) * 32;
    for (int base = 0; base < c.n_run; base += 2 * kSum) {  // warp-uniform
      int e[2] = {-1, -1}, rem[2] = {0, 0};
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = base + u * kSum + t;
        if (j < c.n_run) {
          const int a = c.run_rank[j];
          const int g = c.run_gen[j] + (dec ? 1 : 0);
          if (!dec || g < c.run_out[j]) {  // a decode's finished rows leave (workload.py:134-136)
            int lo = 0, hi = n_est;          // the list is sorted by rank
            while (hi - lo > 1) {
              const int mid = (lo + hi) >> 1;
              if (S.spec_rank[mid] <= a) lo = mid;
              else hi = mid;
            }
            if (!kPart || S.spec_rank[lo] == a) {  // (a partial list holds only the first kSmallEst)
              e[u] = lo;
              rem[u] = S.spec_ol[lo] - g;
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const unsigned peers = __match_any_sync(kFull, e[u]);
        if (e[u] >= 0) {
          const unsigned sum = __reduce_add_sync(peers, (unsigned)rem[u]);
          const unsigned mx = __reduce_max_sync(peers, (unsigned)rem[u]);
          if (lane == __ffs(peers) - 1) {
            atomicAdd(&S.spec_L[e[u]], __popc(peers));
            atomicAdd(&S.spec_rsum[e[u]], (int)sum);
            atomicMax(&S.spec_rmax[e[u]], (int)mx);
          }
        }
      }
    }
    asm volatile("bar.sync 4, %0;" ::"n"((kDWarps - 1) * 32) : "memory");  // warps 1..: summaries complete
    handoff_arrive();  // every input is read: group M may now change the running list, act, q, m
  }
  dphase_mark(c, 19);
  // 2. per-warp metadata (lane e = entry e): PEM segments per entry, with the
  //    running rows as the first segment's prefilled summary
  int nunp = 0, L = 0, base = 0, ol = 0, nj = 0;
  if (lane < n_est) {
    nunp = S.spec_nunp[lane];
    L = S.spec_L[lane];
    base = S.spec_base[lane];
    ol = S.spec_ol[lane];
  }
  int jo = 0, J = 0;
  if (gw > 0) {
    if (lane < n_est) {
      const unsigned tot = (unsigned)(nunp + L);
      nj = tot > 0 ? (int)(((unsigned long long)(tot + (unsigned)pm.mns - 1u) * P.mns_magic) >> 32) : 0;
    }
    const int incl = warp_incl_scan(nj);
    jo = incl - nj;
    J = __shfl_sync(kFull, incl, 31);
  }
  dphase_mark(c, 7);
  // 3. one PEM segment per warp 1..kDWarps-1; the first segment's tok loads
  //    are issued before the barrier, under the RNG replay
  for (int j = gw - 1, first = 1;; j += kDWarps - 1, first = 0) {
    const bool act = gw > 0 && j < J && J <= kMaxJobs;
    int e = 0, k = 0, ne = 0, Le = 0, basee = 0, ole = 0, t0 = 0, nloc = 0;
    int uv[8];
    if (act) {
      const unsigned em = __ballot_sync(kFull, lane < n_est && jo <= j && nj > 0);
      e = 31 - __clz(em);
      k = j - __shfl_sync(kFull, jo, e);
      ne = __shfl_sync(kFull, nunp, e);
      Le = __shfl_sync(kFull, L, e);
      basee = __shfl_sync(kFull, base, e);
      ole = __shfl_sync(kFull, ol, e);
      const int mns = (int)pm.mns;
      t0 = k * mns - Le < 0 ? 0 : k * mns - Le;
      nloc = ((k + 1) * mns - Le < ne ? (k + 1) * mns - Le : ne) - t0;
    }
    const int per = (nloc + 31) >> 5, x0 = lane * per;
#pragma unroll
    for (int i = 0; i < 8; ++i) uv[i] = (act && i < per && x0 + i < nloc) ? T.tok[basee + t0 + x0 + i] : 0;
    if (first) {
      if (gw > 0 && lane == 0 && gw == 1) S.spec_jobs = J;
      GD::sync();
      dphase_mark(c, 20);
      dphase_mark(c, 12);
    }
    if (!act) break;
    const double ratio = S.est_ratio[e];
    int* Uw = S.small.U[gw];
    {
      int ls = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uv[i] = uv[i] ? (int)utok_approx(uv[i], ratio) : 0;
        ls += uv[i];
      }
      int run = warp_incl_scan(ls) - ls;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        run += uv[i];
        if (i < per && x0 + i < nloc) Uw[x0 + i] = run;
      }
    }
    __syncwarp();
    double* tj = S.small.terms + j * kJobTerms;
    double* spill = T.term_spill + (size_t)j * (kSmallMns + 1);
    int nterm = 0, bb = 0, my_end = 0;
    while (bb < nloc) {
      const int before = bb ? Uw[bb - 1] : 0;
      const int ub = Uw[bb];
      const int thr = ub - before > pm.mnbt ? ub : before + (int)pm.mnbt;
      int nb = nloc;
      for (int b2 = bb + 1; b2 < nloc; b2 += 64) {
        const int x = b2 + lane, y = x + 32;
        const bool hx = x < nloc && Uw[x] > thr, hy = y < nloc && Uw[y] > thr;
        const unsigned mx = __ballot_sync(kFull, hx), my = __ballot_sync(kFull, hy);
        if (mx | my) {
          nb = mx ? b2 + __ffs(mx) - 1 : b2 + 32 + __ffs(my) - 1;
          break;
        }
      }
      if (nterm < 32) {
        if (lane == nterm) my_end = nb;
      } else if (lane == 0) {
        const double t = lin(pm.ap, (double)(Uw[nb - 1] - before), pm.bp);
        if (nterm < kJobTerms) tj[nterm] = t;
        else spill[nterm] = t;
      }
      ++nterm;
      bb = nb;
    }
    {
      const int beg = __shfl_up_sync(kFull, my_end, 1);
      if (lane < nterm && lane < 32) {
        const int b0 = lane ? beg : 0;
        tj[lane] = lin(pm.ap, (double)(Uw[my_end - 1] - (b0 ? Uw[b0 - 1] : 0)), pm.bp);
      }
    }
    if (lane == 0) {
      long long rs = (long long)nloc * ole;
      long long mx = nloc > 0 ? ole : 0;
      if (k == 0) {  // the running rows enter the first segment as a prefilled summary
        rs += S.spec_rsum[e];
        mx = S.spec_rmax[e] > mx ? S.spec_rmax[e] : mx;
      }
      const double t = __dadd_rn(__dmul_rn(pm.ad, (double)rs), __dmul_rn(pm.bd, (double)mx));
      if (nterm < kJobTerms) tj[nterm] = t;
      else spill[nterm] = t;
      S.small.nterm[j] = nterm + 1;
    }
    __syncwarp();
  }
  if (gw == 0) {  // warp 0 meanwhile: the entries' segment offsets for the ordered sums
    if (lane < n_est) {  // (the summaries are complete since the barrier above)
      const unsigned tot = (unsigned)(nunp + S.spec_L[lane]);
      nj = tot > 0 ? (int)(((unsigned long long)(tot + (unsigned)pm.mns - 1u) * P.mns_magic) >> 32) : 0;
    }
    const int incl = warp_incl_scan(nj);
    jo = incl - nj;
    if (lane == 0 && S.spec_jobs > kMaxJobs) S.spec_valid = 0;  // did not fit the job buffers
  }
  GD::sync();
  dphase_mark(c, 13);
  if (gw == 0 && lane < n_est && S.spec_jobs <= kMaxJobs) {  // ordered sums, entry by entry, in the reference's order
    double total = 0.0;
    for (int j = jo; j < jo + nj; ++j) {
      const int cj = S.small.nterm[j];
      const double* tj = S.small.terms + j * kJobTerms;
      const int nsm = cj < kJobTerms ? cj : kJobTerms;
      int i = 0;
      for (; i + 4 <= nsm; i += 4) {
        const double2 x = *reinterpret_cast<const double2*>(tj + i);
        const double2 y = *reinterpret_cast<const double2*>(tj + i + 2);
        total = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(total, x.x), x.y), y.x), y.y);
      }
      for (; i < nsm; ++i) total = __dadd_rn(total, tj[i]);
      const double* spill = T.term_spill + (size_t)j * (kSmallMns + 1);
#pragma unroll 1
      for (i = nsm; i < cj; ++i) total = __dadd_rn(total, spill[i]);  // segments of > kJobTerms terms
    }
    S.spec_val[lane] = total;
  }
  dphase_mark(c, 14);
  dphase_mark(c, 21);
}

// After the advance (group D's first warp, behind kBarExecDone; group M is
// already in the next admission): the speculative update becomes this (next)
// iteration's if every chain length it assumed is the advance's; retiring
// relQueries (no unprefilled and no running row left) are not written.  The
// entries kept must be exactly the advance's act list.
template <bool kPart>
__device__ __forceinline__ void spec_commit(Shared& S, const TraceDev& T) {
  Ctl& c = S.c;
  const RqView& rq = S.rq;
  const int lane = threadIdx.x & 31;
  // (c.status may change concurrently: the next admission); a speculated action must be phase E's
  bool ok = S.spec_valid && S.go_exec && S.spec_action == S.action;
#ifdef RS_COUNT_MISSPEC  // experiment: count discarded speculations (phase slot 20)
  if (lane == 0 && S.spec_valid && S.go_exec && S.spec_action != S.action) c.phase[20] += 1;
#endif
  const int n = S.spec_n;
  bool keep = false, bad = false;
  int a = 0;
  if (ok && lane < n) {
    a = S.spec_rank[lane];
    keep = S.spec_nunp[lane] > 0 || S.spec_L[lane] > 0;
    bad = keep && ((S.spec_nunp[lane] > 0 && rq.m[a] != S.spec_m[lane]) ||
                   c.act[__popc(__ballot_sync(__activemask(), keep) & ((1u << lane) - 1u))] != a);
  }
  const unsigned km = __ballot_sync(kFull, keep);
  const int nk = __popc(km);
  // complete: the kept entries are the whole list; partial (the first kSmallEst of a
  // longer list): they are its first nk entries and the next entry lies past them
  const bool tail_ok = kPart && S.spec_part ? nk <= c.n_act && (nk == c.n_act || c.act[nk] > S.spec_rank[n - 1])
                                            : nk == c.n_act;
  ok = ok && !__any_sync(kFull, bad) && tail_ok;
  if (ok && keep) rq.prio[a] = S.spec_val[lane];
  if (lane == 0) {
    if (ok) {
      c.rng = S.spec_rng;
      c.alg_bytes += S.spec_alg;
    }
    S.spec_ok = ok;
    if constexpr (kPart) S.spec_e0 = ok && S.spec_part ? nk : -1;  // where phase B's continuation starts
  }
}


// First sight of this iteration's arrivals [new_lo, new_hi): none of their
// rows is prefilled and their shared chain is not resident (no row of theirs
// was ever inserted), so the sampled uncached-token ratio is exactly 1.0 and
// utok_approx = tok: the estimate is a static function of the trace,
// precomputed at engine creation (first_sight_kernel).  Only the RNG stream
// must advance as the reference's choice() calls would consume it; draws are
// replayed in parallel (jump-ahead) just to detect Lemire rejections, which
// change how many values are consumed (then: sequential replay).
// The generator state after k more next32 values (numpy's half-word buffer:
// a buffered value is consumed first; an odd count leaves a high half buffered).
__device__ __forceinline__ rs_pcg64_state advance32(rs_pcg64_state r, long long k, const JumpEntry* jt) {
  if (k <= 0) return r;
  if (r.has_uint32) {
    r.has_uint32 = 0;
    if (--k == 0) return r;
  }
  const U128 s1 = pcg_jump(U128{r.state_hi, r.state_lo}, (unsigned long long)((k + 1) >> 1), jt);
  r.state_hi = s1.hi;
  r.state_lo = s1.lo;
  r.has_uint32 = (uint32_t)(k & 1);
  r.uinteger = (uint32_t)(pcg_output(s1) >> 32);  // buffered (odd k) or left stale (even k), as numpy does
  return r;
}

__device__ void first_sight(const Params& P, const TraceDev& T, Shared& S, int lo, int hi) {
  Ctl& c = S.c;
  const RqView& rq = S.rq;
  const int tid = threadIdx.x;
  const int Ssz = (int)P.cfg.sample_size;
  for (int a = lo + tid; a < hi; a += kThreads) rq.prio[a] = T.fsprio[a];
  // Replay the draws of arrivals [e_lo, hi) in parallel, each thread a run of
  // stream positions, assuming no Lemire rejection.  A rejection consumes an
  // extra value and shifts every later draw: the arrival that hit the first
  // one is replayed exactly by thread 0 and the parallel replay restarts after it.
  int e_lo = lo;
  while (e_lo < hi) {
    const long long P0 = T.fs_doff[e_lo];
    const long long D = T.fs_doff[hi] - P0;
    if (tid == 0) S.rej_pos = ~0ULL;
    __syncthreads();
    const unsigned h0 = c.rng.has_uint32;
    const U128 s0{c.rng.state_hi, c.rng.state_lo};
    const long long ppt = (D + kThreads - 1) / kThreads;
    long long p = (long long)tid * ppt;
    const long long pend = p + ppt < D ? p + ppt : D;
    if (p < pend) {
      // owner of position p: the last arrival with fs_doff <= P0 + p
      int l = e_lo, r = hi;  // invariant: fs_doff[l] - P0 <= p < fs_doff[r] - P0
      while (r - l > 1) {
        const int mid = (l + r) >> 1;
        if (T.fs_doff[mid] - P0 <= p) l = mid;
        else r = mid;
      }
      int e = l;
      U128 st = s0;
      uint64_t out = 0;
      int half = 0;
      bool fresh = true;
      for (; p < pend; ++p) {
        uint32_t v;
        if (h0 && p == 0) {
          v = c.rng.uinteger;
        } else {
          if (fresh) {
            const long long pp = p - (long long)h0;
            st = pcg_jump(s0, (unsigned long long)(pp >> 1) + 1, S.jt);
            out = pcg_output(st);
            half = (int)(pp & 1);
            fresh = false;
          } else if (half == 0) {
            half = 1;
          } else {
            st = add128(mul128(S.jt[0].a, st), S.jt[0].c);
            out = pcg_output(st);
            half = 0;
          }
          v = half ? (uint32_t)(out >> 32) : (uint32_t)out;
        }
        while (T.fs_doff[e + 1] - P0 <= p) ++e;
        const int d = (int)(p - (T.fs_doff[e] - P0));
        const uint32_t n = (uint32_t)(rq.off[e + 1] - rq.off[e]);
        const uint32_t bound = d < Ssz ? n - (uint32_t)Ssz + (uint32_t)d : (uint32_t)(Ssz - 1 - (d - Ssz));
        const uint32_t excl = bound + 1u;
        const uint32_t left = (uint32_t)((uint64_t)v * excl);
        if (left < excl && left < (0xFFFFFFFFu - bound) % excl) {  // Lemire rejection
          atomicMin(&S.rej_pos, (unsigned long long)p);
          break;
        }
      }
    }
    __syncthreads();
    const unsigned long long rp = S.rej_pos;
    if (rp == ~0ULL) {  // no rejection: consume the D values
      if (tid == 0) c.rng = advance32(c.rng, D, S.jt);
      break;
    }
    if (tid == 0) {  // cold path: the rejecting arrival's choice() call, exactly
      int l = e_lo, r = hi;
      while (r - l > 1) {
        const int mid = (l + r) >> 1;
        if ((unsigned long long)(T.fs_doff[mid] - P0) <= rp) l = mid;
        else r = mid;
      }
      Pcg64 g = Pcg64::from(advance32(c.rng, T.fs_doff[l] - P0, S.jt));
      choice_floyd(g, (uint32_t)(rq.off[l + 1] - rq.off[l]), (uint32_t)Ssz, S.floyd_idx);
      c.rng = g.to();
      S.new_lo_rs = l + 1;
    }
    __syncthreads();
    e_lo = S.new_lo_rs;
  }
  if (tid == 0) c.alg_bytes += 12LL * (hi - lo);  // precomputed priority + draw offset per arrival
  __syncthreads();
}

// General DPU path (first-sight batches of arrivals, many partially
// prefilled relQueries, PEM segments that the token cap can close, or large
// mns / sample sizes): batches of up to kEstBatch relQueries with block scans.
__device__ void dpu_batched(const Params& P, const TraceDev& T, Shared& S, const PemModel& pm) {
  Ctl& c = S.c;
  const RqView& rq = S.rq;
  const rs_config& cfg = P.cfg;
  const int tid = threadIdx.x, lane = tid & 31, warp = opaque_warp();
  const int n_act = c.n_act;
  const int n_new = S.new_hi - S.new_lo;
  const int n_est = n_act + n_new;
  const int Ssz = (int)cfg.sample_size;
  const int dper = 2 * Ssz - 1;  // next32 draws of one choice(n, k=S) call without rejection
  const int batch = kDrawBuf / dper < kEstBatch ? (kDrawBuf / dper > 0 ? kDrawBuf / dper : 1) : kEstBatch;
  const long long B = cfg.block_size;
  if (tid == 0) S.n_est = n_est;

  for (int b0 = 0; b0 < n_est; b0 += batch) {
    const int nb = n_est - b0 < batch ? n_est - b0 : batch;
    // 1. metadata; draw, item and PEM-segment offsets in one block scan
    int dcount = 0, ni = 0, nj = 0;
    if (tid < nb) {
      const int e = b0 + tid;
      const int a = e < n_act ? c.act[e] : S.new_lo + (e - n_act);
      const int off = rq.off[a];
      const int size = rq.off[a + 1] - off;
      const int q = rq.q[a];
      S.est_rank[tid] = a;
      S.est_off[tid] = off;
      S.est_q[tid] = q;
      S.est_nunp[tid] = size - q;
      S.est_ol[tid] = rq.ol[a];
      S.est_m[tid] = rq.m[a];
      dcount = size - q > Ssz ? dper : 0;  // choice() only when k = S < n (prefix_cache.py:157-158)
      ni = size - q;
      const long long tot = (long long)ni + rq.nrun[a];  // running rows enter PEM as a prefilled summary
      nj = tot > 0 ? (int)((tot + pm.mns - 1) / pm.mns) : 0;
    }
    {
      int v[3] = {dcount, ni, nj}, tot[3];
      block_scan32<3>(v, S.s32, tot);
      if (tid < nb) {
        S.est_doff[tid] = v[0] - dcount;
        S.est_io[tid] = v[1] - ni;
        S.est_jo[tid] = v[2] - nj;
      }
      if (tid == 0) {
        S.est_doff[nb] = tot[0];
        S.est_io[nb] = tot[1];
        S.est_jo[nb] = tot[2];
        S.rng_reject = 0;
      }
    }
    __syncthreads();
    const int NI = S.est_io[nb];
    const bool seg = T.seg_ok && NI <= kItemBuf;
    if (tid == 0) c.alg_bytes += 4LL * NI + 4LL * Ssz * (S.est_doff[nb] / dper);  // items' + sampled tok
    // issue the PEM items' tok loads now; they land while the RNG runs
    constexpr int kPer = kItemBuf / kThreads;
    int tokr[kPer];
    int item_e[kPer];
    if (seg) {
      int e = 0;
#pragma unroll
      for (int s = 0; s < kPer; ++s) {
        const int x = s * kThreads + tid;
        tokr[s] = 0;
        item_e[s] = 0;
        if (x < NI) {
          while (S.est_io[e + 1] <= x) ++e;
          item_e[s] = e;
          tokr[s] = T.tok[S.est_off[e] + S.est_q[e] + (x - S.est_io[e])];
        }
      }
    }
    phase_mark(c, 5);
    // 2. numpy's next32 stream, position p -> bounded draw, in parallel
    const int D = S.est_doff[nb];
    const unsigned h0 = c.rng.has_uint32;
    const U128 s0{c.rng.state_hi, c.rng.state_lo};
    {
      const int ppt = (D + kThreads - 1) / kThreads;
      int p = tid * ppt;
      const int pend = p + ppt < D ? p + ppt : D;
      if (p < pend) {
        int e = 0;
        while (S.est_doff[e + 1] <= p) ++e;
        U128 st = s0;
        uint64_t out = 0;
        int half = 0;
        bool fresh = true;
        for (; p < pend; ++p) {
          uint32_t v;
          if (h0 && p == 0) {
            v = c.rng.uinteger;
          } else {
            if (fresh) {
              const long long pp = p - (long long)h0;
              st = pcg_jump(s0, (unsigned long long)(pp >> 1) + 1, S.jt);
              out = pcg_output(st);
              half = (int)(pp & 1);
              fresh = false;
            } else if (half == 0) {
              half = 1;
            } else {
              st = add128(mul128(S.jt[0].a, st), S.jt[0].c);
              out = pcg_output(st);
              half = 0;
            }
            v = half ? (uint32_t)(out >> 32) : (uint32_t)out;
          }
          while (S.est_doff[e + 1] <= p) ++e;
          const int d = p - S.est_doff[e];
          const uint32_t nunp = (uint32_t)S.est_nunp[e];
          // Floyd draws bounded(j), j = n-k .. n-1, then the shuffle's bounded(i), i = k-1 .. 1
          const uint32_t bound = d < Ssz ? nunp - (uint32_t)Ssz + (uint32_t)d : (uint32_t)(Ssz - 1 - (d - Ssz));
          const uint32_t excl = bound + 1u;
          const uint64_t mm = (uint64_t)v * excl;
          const uint32_t left = (uint32_t)mm;
          if (left < excl && left < (0xFFFFFFFFu - bound) % excl) S.rng_reject = 1;  // Lemire rejection
          S.draws[p] = (uint32_t)(mm >> 32);
        }
      }
    }
    __syncthreads();
    phase_mark(c, 6);
    // 3. sample ratios
    if (S.rng_reject) {  // a rejection shifts the stream: replay this batch sequentially
      if (tid == 0) {
        Pcg64 g = Pcg64::from(c.rng);
        for (int e = 0; e < nb; ++e) S.est_ratio[e] = sample_ratio_seq(g, T, rq, P, S.est_rank[e], S.floyd_idx);
        c.rng = g.to();
      }
    } else {
      if (tid < nb) {
        const int nunp = S.est_nunp[tid];
        const int base = S.est_off[tid] + S.est_q[tid];
        const long long mh = B * (long long)S.est_m[tid];  // exact utok = tok - B*m
        double ratio = 0.0;
        if (nunp > 0) {
          long long usum = 0, tsum = 0;
          if (nunp <= Ssz) {
            for (int i = 0; i < nunp; ++i) {
              const long long t = T.tok[base + i];
              usum += t - mh;
              tsum += t;
            }
          } else if (Ssz <= 16) {  // Floyd's set in registers; the shuffle only permutes it
            const int d0 = S.est_doff[tid];
            uint32_t idx[16];
#pragma unroll
            for (int d = 0; d < 16; ++d) {
              if (d < Ssz) {
                const uint32_t j = (uint32_t)(nunp - Ssz + d);
                const uint32_t v = S.draws[d0 + d];
                bool found = false;
#pragma unroll
                for (int x = 0; x < 16; ++x) found |= (x < d) && idx[x] == v;
                idx[d] = found ? j : v;
              }
            }
            long long tv[16];
#pragma unroll
            for (int d = 0; d < 16; ++d) tv[d] = d < Ssz ? T.tok[base + (int)idx[d]] : 0;
#pragma unroll
            for (int d = 0; d < 16; ++d)
              if (d < Ssz) {
                usum += tv[d] - mh;
                tsum += tv[d];
              }
          } else {
            uint32_t idx[kMaxSample];
            const int d0 = S.est_doff[tid];
            for (int d = 0; d < Ssz; ++d) {
              const uint32_t j = (uint32_t)(nunp - Ssz + d);
              const uint32_t v = S.draws[d0 + d];
              bool found = false;
              for (int x = 0; x < d; ++x) found |= idx[x] == v;
              idx[d] = found ? j : v;
            }
            for (int d = 0; d < Ssz; ++d) {
              const long long t = T.tok[base + (int)idx[d]];
              usum += t - mh;
              tsum += t;
            }
          }
          ratio = __ddiv_rn((double)usum, (double)tsum);
        }
        S.est_ratio[tid] = ratio;
      }
      if (tid == 0 && D > 0) {  // advance the generator past the D values
        const long long cnt = (long long)D - (long long)h0;
        if (cnt <= 0) {
          c.rng.has_uint32 = 0;
        } else {
          const U128 s1 = pcg_jump(s0, (unsigned long long)((cnt + 1) >> 1), S.jt);
          c.rng.state_hi = s1.hi;
          c.rng.state_lo = s1.lo;
          c.rng.has_uint32 = (uint32_t)(cnt & 1);
          c.rng.uinteger = (uint32_t)(pcg_output(s1) >> 32);  // numpy leaves it stale when consumed
        }
      }
    }
    // running rows of each relQuery enter PEM as a prefilled summary (count,
    // sum and max of remaining): they precede the unprefilled rows and fit
    // the first segment (running <= mns)
    for (int eb = warp; eb < nb; eb += kWarps) {
      const int a = S.est_rank[eb];
      const int ol = S.est_ol[eb];
      PrefixSummary ps{0, 0, 0};
      if (S.est_q[eb] > 0) {
        long long rs = 0, cnt = 0, mx = 0;
        for (int j = lane; j < c.n_run; j += 32)
          if (c.run_rank[j] == a) {
            const long long r = ol - c.run_gen[j];
            rs += r;
            cnt += 1;
            mx = r > mx ? r : mx;
          }
        ps.n = (int)warp_sum(cnt);
        ps.rsum = warp_sum(rs);
        ps.rmax = (int)warp_max(mx);
      }
      if (lane == 0) S.est_ps[eb] = ps;
    }
    __syncthreads();
    phase_mark(c, 7);
    // 4. PEM
    if (seg) {
      SegBuf sb{S.seg.U, S.seg.UNP, S.seg.REM, S.seg.terms, S.seg.jcnt, S.est_io, S.est_jo};
      // each thread materialises exactly the items whose tok it loaded
      long long carryU = 0, carryN = 0;
#pragma unroll
      for (int s = 0; s < kPer; ++s) {
        const int x = s * kThreads + tid;
        if (s * kThreads < NI) {
          int u = 0;
          if (x < NI) {
            u = (int)utok_approx(tokr[s], S.est_ratio[item_e[s]]);
            S.seg.REM[x] = S.est_ol[item_e[s]];
          }
          int v[2] = {u, x < NI ? 1 : 0}, tot[2];
          block_scan32<2>(v, S.s32, tot);
          if (x < NI) {
            S.seg.U[x] = carryU + v[0];
            S.seg.UNP[x] = (int)(carryN + v[1]);
          }
          carryU += tot[0];
          carryN += tot[1];
        }
      }
      __syncthreads();
      seg_jobs_and_sum(nb, S.est_ps, pm, sb, PrioOut{rq.prio, S.est_rank});
    } else {
      for (int eb = warp; eb < nb; eb += kWarps) {
        UnprefItems it{T.tok, S.est_off[eb] + S.est_q[eb], S.est_ol[eb], S.est_ratio[eb]};
        const double v = warp_pem(it, S.est_nunp[eb], S.est_ps[eb], pm);
        if (lane == 0) rq.prio[S.est_rank[eb]] = v;
      }
      __syncthreads();
    }
    phase_mark(c, 8);
  }
}

// e_start: the first entry of the re-estimate list to estimate (> 0 after a
// partial speculative update, which covered the entries before it).
template <bool kFast, bool kC, bool kPart = false>
__device__ void dpu_update(const Params& P, const TraceDev& T, Shared& S, const int e_start = 0) {
  Ctl& c = S.c;
  const RqView& rq = S.rq;
  const rs_config& cfg = P.cfg;
  const int tid = threadIdx.x;
  PemModel pm;
  pm.ap = P.pol.alpha_p;
  pm.bp = P.pol.beta_p;
  pm.ad = P.pol.alpha_d;
  pm.bd = P.pol.beta_d;
  pm.cap = cfg.cap;
  pm.mns = cfg.max_num_seqs;
  pm.mnbt = cfg.max_num_batched_tokens;
  if constexpr (kFast) {
    // partially prefilled relQueries (in rank order), then the arrivals
    const int n_act = c.n_act;
    for (int e0 = kPart ? e_start : 0; e0 < n_act;) {
      e0 += dpu_small<kC>(P, T, S, pm, e0, n_act);
      __syncthreads();
    }
    if (S.new_hi > S.new_lo) first_sight(P, T, S, S.new_lo, S.new_hi);
    if (tid == 0) S.n_est = n_act + (S.new_hi - S.new_lo);
  } else {
    dpu_batched(P, T, S, pm);
  }
  // starvation override (priority.py:318-339): wholly waiting = no prefilled row = q == 0
  if (!kC && isfinite(cfg.tau)) {
    for (int a = tid; a < c.n_admitted; a += kThreads) {
      const int size = rq.off[a + 1] - rq.off[a];
      if (rq.q[a] == 0 && size > 0) {
        const double uw = __ddiv_rn(__dsub_rn(c.clock, rq.arrival[a]), (double)size);
        if (uw > cfg.tau) rq.prio[a] = 0.0;
      }
    }
    __syncthreads();
  }
  // (every estimating path above ends with a barrier: the waiting order sees the new values)
}

}  // namespace rsd
