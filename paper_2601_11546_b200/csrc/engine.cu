// engine.cu -- the RelServe scheduler loop as one persistent sm_100a CTA per trace.
//
// Replaces the reference's per-iteration Python loops (Engine.run,
// pkg/src/relsim/engine.py:371-448).  Each CTA owns one trace and runs up to
// `max_iters` scheduler iterations per launch with no host round trip:
//
//   A  admission                      engine.py:243-269
//   B  Dynamic Priority Updater       priority.py:261-339        (dpu.cuh)
//   C  waiting-queue order: top-1     engine.py:277-281: key (prio, arrival,
//      over a static order + the      rel_id) == (prio bits, admission rank);
//      re-estimated relQueries;       sharded pool: allgather of the shards'
//      waiting count                  heads and priorities (shard.cuh)
//   D  candidates                     engine.py:285-308, arranger.py:71-112
//   E  decision + Delta projection    engine.py:387-433, arranger.py:115-179
//   F  state advance                  engine.py:315-363, 439-448, with the
//                                     prefix-cache model (cache_model.cuh)
//
// Device layout: engine_state.cuh.  The control block (clock, running list
// with its rows' state, queues, RNG, cache bookkeeping) and, when it fits,
// the relQuery table live in shared memory for the whole launch; request rows
// stay in HBM and are touched only for re-estimated relQueries, candidate
// rows and completions.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cstddef>
#include <cstdlib>
#include <functional>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/relserve.h"

#ifndef RS_PREFETCH_HEAD
#define RS_PREFETCH_HEAD 1  // the previous head's next candidate rows, prefetched into L1 during the DPU
#endif
#include "cache_model.cuh"
#include "dpu.cuh"
#include "engine_state.cuh"
#include "radix_sort.cuh"
#include "shard.cuh"

namespace rsd {

// ---------------------------------------------------------------------------
// One scheduler iteration (all threads).  Returns false when the trace stopped.
// ---------------------------------------------------------------------------

// The Adaptive Batch Arranger's decision, thread 0 (engine.py:387-433):
// project_delta (arranger.py:115-143) when both candidates are non-empty and
// m+ <= m-, evaluated left to right in fp64 exactly as written, then
// decide_next (arranger.py:146-179); fcfs/sp are prefill-first
// (engine.py:387-395).  ol(i) is the output limit of the i-th distinct
// running relQuery in rel_id order (engine.py:406-408); internal = the first
// running row attaining m+ belongs to the prefill candidate's relQuery.
// Outputs follow rs_iter_record: NaN where the reference logs None.
// Proj supplies the projection's per-relQuery terms: term(i, adn, ol_p) =
// (alpha_d * n_p) * min(OL_i, OL_p) of the i-th distinct running relQuery in
// rel_id order, and max_ol(n) = max OL over them (the engine precomputes both in
// parallel; the unit entry point computes them here).
template <class Proj>
__device__ __forceinline__ void arrange(const rs_cost_model& m, bool prefill_first, int force, bool has_p,
                                        bool has_d, bool internal, double m_plus, double m_minus, long long utok_sum,
                                        int n_p, long long ol_p, int n_dist, const Proj& pj, long long W, int& action,
                                        int& kase, double& mp, double& mmn, double& dp, double& dm, double& dt) {
  dp = dm = dt = __longlong_as_double(0x7FF8000000000000LL);
  mp = m_plus;
  mmn = m_minus;
  if (prefill_first) {
    kase = RS_CASE_FORCED;
    if (has_p) action = RS_ACTION_PREFILL;
    else if (has_d) action = RS_ACTION_DECODE;
    else {
      action = RS_ACTION_IDLE;
      mp = mmn = dp;
    }
    return;
  }
  double ddp = 0, ddm = 0, ddt = 0;
  // project_delta: the reference also evaluates it for internal decisions
  // (engine.py:397-415), but only the transitional case reads it (arranger.py:146-179)
  if (has_p && has_d && !internal && m_plus <= m_minus) {
    const double l_prefill = __dadd_rn(__dmul_rn(m.alpha_p, (double)utok_sum), m.beta_p);
    ddp = __dmul_rn(l_prefill, (double)n_dist);
    const double adn = __dmul_rn(m.alpha_d, (double)n_p);
    int i = 0;
    for (; i + 4 <= n_dist; i += 4) {  // the adds stay in order; the terms are independent
      const double t0 = pj.term(i, adn, ol_p), t1 = pj.term(i + 1, adn, ol_p), t2 = pj.term(i + 2, adn, ol_p),
                   t3 = pj.term(i + 3, adn, ol_p);
      ddp = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(ddp, t0), t1), t2), t3);
    }
#pragma unroll 1
    for (; i < n_dist; ++i) ddp = __dadd_rn(ddp, pj.term(i, adn, ol_p));
    const long long max_ol = pj.max_ol(n_dist);
    ddm = -__dmul_rn(__dmul_rn((double)W, m.beta_d), (double)(ol_p < max_ol ? ol_p : max_ol));
    ddt = __dadd_rn(ddp, ddm);
  }
  if (!has_p && !has_d) {
    action = RS_ACTION_IDLE;
    kase = RS_CASE_FORCED;
    mp = mmn = dp;
  } else if (!has_d) {
    action = RS_ACTION_PREFILL;
    kase = RS_CASE_FORCED;
  } else if (!has_p) {
    action = RS_ACTION_DECODE;
    kase = RS_CASE_FORCED;
  } else if (internal) {
    action = RS_ACTION_PREFILL;
    kase = RS_CASE_INTERNAL;
  } else if (m_plus > m_minus) {
    action = RS_ACTION_PREFILL;
    kase = RS_CASE_PREEMPT;
  } else {
    kase = RS_CASE_TRANSITIONAL;
    dp = ddp;
    dm = ddm;
    dt = ddt;
    if (force == 1) action = RS_ACTION_PREFILL;
    else if (force == 2) action = RS_ACTION_DECODE;
    else action = (ddt < 0) ? RS_ACTION_PREFILL : RS_ACTION_DECODE;
  }
}

struct OlProj {  // rs_arrange: terms from the sorted output limits
  const long long* ol;
  __device__ __forceinline__ double term(int i, double adn, long long ol_p) const {
    return __dmul_rn(adn, (double)(ol[i] < ol_p ? ol[i] : ol_p));
  }
  __device__ __forceinline__ long long max_ol(int n) const {
    long long x = 0;
    for (int i = 0; i < n; ++i) x = ol[i] > x ? ol[i] : x;
    return x;
  }
};
struct TermProj {  // the engine: terms precomputed by the whole CTA (phase E)
  const double* t;
  long long mx;
  __device__ __forceinline__ double term(int i, double, long long) const { return t[i]; }
  __device__ __forceinline__ long long max_ol(int) const { return mx; }
};

// Parity mode: snapshot of this iteration's priority update into row `row`
// (all threads): every admitted relQuery's priority and flags (estimated /
// starvation override / live / waiting) and the DPU generator state -- the
// reference's PriorityRecord per live relQuery (priority.py:287-315) and the
// generator state after update().  The waiting order (engine.py:277-281) is
// derived from it after the launch by the radix sort (rs_engine_read_order):
// the timed path never sorts.
__device__ __noinline__ void record_parity(const Params& P, const TraceDev& T, Shared& S, long long row) {
  const Ctl& c = S.c;
  const RqView& rq = S.rq;
  const rs_config& cfg = P.cfg;
  double* vp = T.snap_prio + (size_t)row * T.R;
  unsigned char* fp = T.snap_flag + (size_t)row * T.R;
  const bool dpu = P.use_dpu;
  const bool tau_on = dpu && isfinite(cfg.tau);
  for (int a = threadIdx.x; a < T.R; a += kThreads) {
    unsigned char f = 0;
    double v = qnan();
    if (a < c.n_admitted) {
      const int size = rq.off[a + 1] - rq.off[a];
      v = rq.prio[a];
      if (rq.ndone[a] < size || size == 0) f |= kSnapLive;
      if (rq.q[a] < size) f |= kSnapWaiting;
      if (dpu && a >= S.new_lo && a < S.new_hi) f |= kSnapEstimated;  // first sight
      if (tau_on && rq.q[a] == 0 && size > 0 &&
          __ddiv_rn(__dsub_rn(c.clock, rq.arrival[a]), (double)size) > cfg.tau)
        f |= kSnapOverride;
    }
    vp[a] = v;
    fp[a] = f;
  }
  __syncthreads();
  if (dpu)  // the re-estimated partially prefilled relQueries (every shard's, in a sharded pool)
    for (int j = threadIdx.x; j < c.n_act; j += kThreads) fp[c.act[j]] |= kSnapEstimated;
  if (threadIdx.x == 0) T.snap_rng[row] = c.rng;
  __syncthreads();
}

// _world_duration (engine.py:310-313): base * (1 + sigma * z), clamped at 0,
// z = the n-th standard normal of the engine's noise stream (one per executed batch)
template <bool kC>
__device__ __forceinline__ double world_duration(const Params& P, const TraceDev& T, long long n, double base) {
  if (!kC && P.cfg.noise_sigma > 0) {
    const double v = __dmul_rn(base, __dadd_rn(1.0, __dmul_rn(P.cfg.noise_sigma, T.noise[n])));
    base = v > 0.0 ? v : 0.0;  // max(0.0, v)
  }
  return base;
}

// ---- F: execute the decided action (engine.py:315-363, 435-448) on warp
// group G (the whole CTA, or group M of the pipelined common-configuration
// iteration, which waits at the handoff barrier (kHand) before its first write
// of state group D reads).  Returns false when the trace stopped.
template <bool kC, class G, bool kHand>
__device__ __forceinline__ bool execute(const Params& P, const TraceDev& T, Shared& S, const int action) {
  Ctl& c = S.c;
  const RqView& rq = S.rq;
  const int tid = threadIdx.x;
  const rs_config& cfg = P.cfg;
  if (action == RS_ACTION_PREFILL) {  // _execute_prefill (engine.py:315-341)
    const int h = S.head;
    const int q = rq.q[h];
    const int row0 = rq.off[h] + q;
    const int n = S.taken;
    const int n_run0 = c.n_run;
    const int ol = rq.ol[h];
    // read before the cache advance (nothing in this iteration changes them before thread 0's
    // bookkeeping): their latency -- HBM when the relQuery table does not fit in shared
    // memory -- overlaps the advance instead of thread 0's serial section
    const int size_h = rq.off[h + 1] - rq.off[h];
    const int nrun_h = rq.nrun[h];
    long long ut = 0;
    const bool fast = prefill_fast<kC, G, kHand>(P, T, S, h, n, S.cand_tok, ut);
    if (kHand && !fast) handoff_wait();  // the exact per-row path changes rq.m too
    phase_mark(c, 9);
    if (tid == 0) {
      bool ok = c.status == RS_RUNNING;
      if (!fast && ok) {
        for (int i = 0; i < n; ++i) {
          const long long u = prefill_row_cache(c, T, rq, P, h, S.cand_tok[i]);
          if (u < 0) {
            ok = false;
            break;
          }
          ut += u;
        }
      }
      if (ok) {
        c.alg_bytes += 16LL * n;  // FIFO pushes (window reads are counted in prefill_fast)
        const double start = c.clock;
        const double dur =
            world_duration<kC>(P, T, c.n_batch++, __dadd_rn(__dmul_rn(P.world.alpha_p, (double)ut), P.world.beta_p));
        c.n_run = n_run0 + n;
        rq.q[h] = q + n;
        if (h == c.zh_idx) c.zh_valid = 0;  // the cached static-order head may have left the order
        if (q + n == size_h) c.n_wait--;  // no pending rows left: leaves waiting
        if (nrun_h == 0) c.rrq[c.n_rrq++] = h;
        rq.nrun[h] = nrun_h + n;
        if (q == 0 && (kC || P.use_dpu)) {  // becomes partially prefilled: join the re-estimate list
          int pos = c.n_act;
          if (pos >= kMaxAct) {
            c.status = RS_EUNSUPPORTED;
            c.error_detail = 3;
          } else {
            while (pos > 0 && c.act[pos - 1] > h) {
              c.act[pos] = c.act[pos - 1];
              --pos;
            }
            c.act[pos] = h;
            c.n_act++;
          }
        }
        c.clock = __dadd_rn(c.clock, dur);
        if (q == 0) T.fps[h] = start;  // first_prefill_start is set once (engine.py:338-339)
        T.lpe[h] = c.clock;
        if (kC || (cfg.log_decisions && T.log_cap > 0)) {
          rs_iter_record& r = T.log[c.n_log & (T.log_cap - 1)];
          r.batch_rq = h;
          r.batch_first = q;
          r.batch_n = n;
        }
      }
      S.go = ok && c.status == RS_RUNNING;
    }
    // running list append + kv reservation (engine.py:326-329): sum of
    // (tok + output_limit) = candidate kv prefix at n-1
    for (int i = tid; i < n; i += G::kN) {
      c.run_row[n_run0 + i] = row0 + i;
      c.run_rank[n_run0 + i] = h;
      c.run_gen[n_run0 + i] = 0;
      c.run_out[n_run0 + i] = S.cand_out[i];
      c.run_kv[n_run0 + i] = S.cand_tok[i] + ol;
    }
    if (tid == 0) c.kv += (long long)S.cand_u[n - 1] + (long long)n * (S.cand_mh + ol);
    G::sync();
    phase_mark(c, 10);
    if (!S.go) return false;
  } else if (action == RS_ACTION_DECODE) {  // _execute_decode (engine.py:343-363)
    const int n = c.n_run;
    if (tid == 0) {
      S.act_dirty = 0;
      S.rrq_dirty = 0;
    }
    G::sync();
    const double clk = __dadd_rn(
        c.clock, world_duration<kC>(P, T, c.n_batch, __dadd_rn(__dmul_rn(P.world.alpha_d, (double)n), P.world.beta_d)));
    int kv_free = 0;
    int keep[kMaxRun / G::kN], nrow[kMaxRun / G::kN], nrank[kMaxRun / G::kN];
    int ngen[kMaxRun / G::kN], nout[kMaxRun / G::kN], nkv[kMaxRun / G::kN];
#pragma unroll
    for (int s = 0; s < kMaxRun / G::kN; ++s) {
      const int j = s * G::kN + tid;
      keep[s] = 0;
      if (j < n) {
        const int r = c.run_row[j];
        const int a = c.run_rank[j];
        const int g = c.run_gen[j] + 1;
        nrow[s] = r;
        nrank[s] = a;
        ngen[s] = g;
        nout[s] = c.run_out[j];
        nkv[s] = c.run_kv[j];
        if (g >= nout[s]) {  // done (workload.py:134-136)
          T.gen[r] = g;
          T.comp[r] = (int)c.iteration;
          kv_free += nkv[s];
          const int nrun_old = atomicSub(&rq.nrun[a], 1);  // both in flight at once
          const int ndone_old = atomicAdd(&rq.ndone[a], 1);
          if (nrun_old == 1) S.rrq_dirty = 1;
          if (ndone_old + 1 == rq.off[a + 1] - rq.off[a]) {
            T.lde[a] = clk;  // relQuery retired (engine.py:360-362)
            atomicSub(&c.live, 1);
            S.act_dirty = 1;
          }
        } else {
          keep[s] = 1;
        }
      }
    }
    // stable compaction of the running list + freed kv, one fused scan per
    // tile (the scan's first barrier orders all reads of the old list)
    if constexpr (kHand) handoff_wait();  // group D has read the running list and the act list
    int cbase = 0;
    long long kv_total = 0;
#pragma unroll
    for (int s = 0; s < kMaxRun / G::kN; ++s) {
      if (s * G::kN < n) {
        int v[2] = {keep[s], (int)kv_free}, tot[2];
        kv_free = 0;
        group_scan32<G, 2>(v, S.s32, tot, tid >> 5);
        if (keep[s]) {
          const int d = cbase + v[0] - 1;
          c.run_row[d] = nrow[s];
          c.run_rank[d] = nrank[s];
          c.run_gen[d] = ngen[s];
          c.run_out[d] = nout[s];
          c.run_kv[d] = nkv[s];
        }
        cbase += tot[0];
        kv_total += tot[1];
      }
    }
    G::sync();
    if (opaque_warp() == 0) {
      // warp 0: the distinct running relQueries without running rows leave rrq, retired
      // relQueries the re-estimate list (stable compactions, 32 entries per round: the
      // relQuery table may sit in HBM, where a serial loop pays a load latency per entry)
      if (S.rrq_dirty) {
        const int w = warp_compact(c.rrq, c.n_rrq, [&](int a) { return rq.nrun[a] > 0; });
        if (opaque_lane() == 0) c.n_rrq = w;
      }
      if (S.act_dirty && (kC || P.use_dpu)) {
        const int w = warp_compact(c.act, c.n_act, [&](int a) { return rq.ndone[a] < rq.off[a + 1] - rq.off[a]; });
        if (opaque_lane() == 0) c.n_act = w;
      }
    }
    if (tid == 0) {
      c.alg_bytes += 8LL * (n - cbase);  // generated + completion iteration of finished rows
      c.n_run = cbase;
      c.kv -= kv_total;
      c.clock = clk;
      c.n_batch++;
      if (kC || (cfg.log_decisions && T.log_cap > 0)) T.log[c.n_log & (T.log_cap - 1)].batch_n = n;
    }
  } else {  // idle (engine.py:439-447)
    if constexpr (kHand) handoff_wait();
    if (tid == 0) {
      if (c.n_admitted >= T.R) {
        c.status = c.live ? RS_EABORT_IDLE : RS_OK;
        S.go = 0;
        if (kC || (cfg.log_decisions && T.log_cap > 0)) {
          T.log[c.n_log & (T.log_cap - 1)].kv_reserved = c.kv;
          c.n_log++;
        }
      } else {
        const double nxt = rq.arrival[c.n_admitted];
        if (nxt > c.clock) c.clock = nxt;
        S.go = 1;
      }
    }
    G::sync();
    if (!S.go) return false;
  }
  if (tid == 0) {
    if (kC || (cfg.log_decisions && T.log_cap > 0)) {
      T.log[c.n_log & (T.log_cap - 1)].kv_reserved = c.kv;
      c.n_log++;
    }
    c.iteration++;
    S.pf_head = S.head;  // read after the next admission barrier
  }
  phase_mark(c, 4);
  // no closing barrier: the next admission (thread 0) touches nothing the other threads
  // still read here (its flag is S.go_admit, not the execution phase's S.go)
  return true;
  return true;
}

// The prefill candidate's scan (arranger.py:80-112) over the head h's pending rows:
// S.cand_tok / cand_out / cand_u (inclusive utok prefix) and S.first_bad, the first
// row that breaks a constraint (S.first_bad must be 0x7FFFFFFF on entry); J = the rows
// scanned at most, mh = B * resident chain blocks of h.  All threads of group G.
template <bool kC, class G>
__device__ __forceinline__ void cand_scan(const Params& P, const TraceDev& T, Shared& S, const int h, int& J,
                                          int& mh) {
  const Ctl& c = S.c;
  const RqView& rq = S.rq;
  const rs_config& cfg = P.cfg;
  const int tid = threadIdx.x;
  int base_row = 0, olh = 0;
  J = 0;
  mh = 0;
  if (h >= 0) {
    const int q = rq.q[h];
    base_row = rq.off[h] + q;
    const int pend = rq.off[h + 1] - base_row;
    const long long room = cfg.max_num_seqs - c.n_run;
    J = room <= 0 ? 0 : (int)(pend < room ? pend : room);
    mh = (int)((kC ? 16 : cfg.block_size) * (long long)rq.m[h]);
    olh = rq.ol[h];
  }
  const long long headroom = cfg.cap - c.kv;
  int cu = 0, ck = 0;
  for (int base = 0; base < J; base += G::kN) {
    const int j = base + tid;
    int v[2] = {0, 0};
    if (j < J) {
      const int t = T.tok[base_row + j];
      S.cand_tok[j] = t;
      S.cand_out[j] = T.out[base_row + j];
      v[0] = t - mh;   // exact utok (match_uncached, refresh=False)
      v[1] = t + olh;  // kv need
    }
    int tot[2];
    group_scan32<G, 2>(v, S.s32, tot, tid >> 5);
    bool bad = false;
    if (j < J) {
      const int U = cu + v[0], K = ck + v[1];
      S.cand_u[j] = U;
      bad = (j > 0 && U > cfg.max_num_batched_tokens) || K > headroom;
    }
    const unsigned m = __ballot_sync(kFull, bad);
    if (m && (tid & 31) == 0) atomicMin(&S.first_bad, base + (tid & ~31) + __ffs(m) - 1);
    cu += tot[0];
    ck += tot[1];
    G::sync();
    if (S.first_bad < J) break;
  }
}

// kC: the common configuration, fixed at compile time (a DPU policy, tau = inf,
// no world-model noise, one shard, decision log on,
// the default block size 16 and sample size 8):
// the checks for everything else leave the iteration's instruction stream.
template <bool kFast, bool kC, bool kPart>
__device__ bool iterate(const Params& P, const TraceDev& T, Shared& S, const bool last) {
  Ctl& c = S.c;
  const RqView& rq = S.rq;
  const int tid = threadIdx.x;
  const rs_config& cfg = P.cfg;

  // ---- A: termination + admission (engine.py:375-380, 243-269)
  if (tid == 0) {
    S.go_admit = 1;
    if (c.live == 0 && c.n_admitted == T.R) {
      c.status = RS_OK;
      S.go_admit = 0;
    } else if (c.iteration >= cfg.iteration_limit) {
      c.status = RS_EABORT_LIMIT;
      S.go_admit = 0;
    } else if (!kC && cfg.noise_sigma > 0 && c.n_batch >= T.noise_n) {
      S.go_admit = 0;  // out of noise draws: end the launch, still running (the host appends more)
    } else {
      // admission ranks are sorted by arrival: gallop, then bisect, to the first arrival > clock
      const int a0 = c.n_admitted;
      int a = a0;
      if (a < T.R && rq.arrival[a] <= c.clock) {
        int lo_a = a, step = 1;  // arrival[lo_a] <= clock
        while (a + step < T.R && rq.arrival[a + step] <= c.clock) {
          lo_a = a + step;
          step <<= 1;
        }
        int hi_a = a + step < T.R ? a + step : T.R;  // arrival[hi_a] > clock, or the end
        while (hi_a - lo_a > 1) {
          const int mid = (lo_a + hi_a) >> 1;
          if (rq.arrival[mid] <= c.clock) lo_a = mid;
          else hi_a = mid;
        }
        a = hi_a;
        c.n_wait += T.ne_pref[a] - T.ne_pref[a0];  // waiting entries: the arrivals with rows
        c.zh_valid = 0;                             // they may precede the cached static-order head
      }
      c.live += a - a0;
      c.n_admitted = a;
      S.new_lo = a0;
      S.new_hi = a;
    }
  }
  __syncthreads();
  if (!S.go_admit) return false;
  phase_mark(c, 0);
#if RS_PREFETCH_HEAD
  if (tid >= kThreads - 32) {  // the last warp: pull the previous head's next candidate rows into L1
    int h = S.pf_head;
    const int l = tid & 31;
    if constexpr (kPart) {  // large traces: a fully prefilled head is followed by the static order's next entry
      if (h >= 0 && rq.q[h] >= rq.off[h + 1] - rq.off[h]) {
        const int z = c.zptr + (rq.zl[c.zptr < T.nzl ? c.zptr : 0] == h ? 1 : 0);
        h = z < T.nzl ? rq.zl[z] : -1;
      }
    }
    if (h >= 0 && l < 18) {
      const int lo = rq.off[h] + rq.q[h], hi = rq.off[h + 1];
      const int r = lo + (l % 9) * 32;  // 9 lines of 128 B cover the <= 256 rows of a candidate
      if (r < hi) {
        const int* p = (l < 9 ? T.tok : T.out) + r;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
      }
    }
  }
#endif

  // ---- B: priorities.  fcfs: 0.0; sp: static_relquery_prio, both set at
  // admission (engine.py:255-267, preloaded into prio); relserve*: the DPU.
  if constexpr (kC) {
    // the launch's first iteration, the speculative update was not usable, or (kPart) it
    // covered a prefix of the list only
    if (!S.spec_ok || (kPart && S.spec_e0 >= 0)) {
      if constexpr (kPart) dpu_update<kFast, kC, true>(P, T, S, S.spec_ok ? S.spec_e0 : 0);
      else dpu_update<kFast, kC>(P, T, S);
    } else {  // the re-estimates were computed during the previous advance: only the arrivals remain
      if (S.new_hi > S.new_lo) first_sight(P, T, S, S.new_lo, S.new_hi);
      if (tid == 0) S.n_est = c.n_act + (S.new_hi - S.new_lo);
    }
  } else if (P.use_dpu) {
    dpu_update<kFast, kC>(P, T, S);
  } else if (tid == 0) {
    S.n_est = 0;
  }
  phase_mark(c, 1);

  // kC: group D leaves the iteration here.  The waiting order, the candidates
  // and the decision run on group M alone; group D computes the next
  // iteration's update from the state this iteration's action will leave --
  // at once when the action is already certain (a decode forced by a full
  // running set or an empty waiting queue: no prefill candidate can exist,
  // arranger.py:80-112, 146-179), else once group M has the candidates
  // (kBarDecision).
  const bool early = c.n_run > 0 && (c.n_run >= cfg.max_num_seqs || c.n_wait == 0);
  if constexpr (kC) {
    if (opaque_warp() >= kMWarps) {
      if (T.snap_prio) record_parity(P, T, S, c.n_log & (T.log_cap - 1));  // meets group M's call (whole CTA)
      const bool allowed = !last && c.iteration + 1 < cfg.iteration_limit;
      int action = RS_ACTION_DECODE, h = -1, nh = 0;
      if (!early) {  // once the candidates are known, decide_next (arranger.py:146-179) as far as
        decision_wait();  // it goes without the Delta projection: no prefill candidate -> decode (or
        h = S.head;       // idle); internal or preemption -> prefill; transitional: forced by the
        nh = S.taken;     // policy, else the prefill is speculated (spec_commit discards the update
        if (nh == 0) {    // if phase E decided otherwise; never at configs 2, 3 and 5)
          action = c.n_run > 0 ? RS_ACTION_DECODE : RS_ACTION_IDLE;
        } else if (c.n_run == 0 || S.dmin_slot == h || S.m_plus > S.m_minus) {
          action = RS_ACTION_PREFILL;
        } else {
          action = P.force == 2 ? RS_ACTION_DECODE : RS_ACTION_PREFILL;
        }
      }
      if ((threadIdx.x & 31) == 0 && opaque_warp() == kMWarps) S.spec_action = action;
      dpu_spec<kPart>(P, T, S, action, h, nh, allowed);
      exec_done_wait();
      if (opaque_warp() == kMWarps) spec_commit<kPart>(S, T);
      return S.go_exec;
    }
  }
  // the threads and barrier of phases C-E: the whole CTA, or group M (kC)
  using GC = typename std::conditional<kC, GM, GAll>::type;
  constexpr int NT = GC::kN;

  // ---- C: waiting head = argmin (prio, rank) over relQueries with pending
  // rows, and W = len(waiting) (engine.py:277-281).  A relQuery none of whose
  // rows was prefilled keeps a static priority (first-sight estimate reused,
  // priority.py:261-266, 298-302; sp/fcfs: fixed at admission), so those are
  // visited in a precomputed (priority bits, rank) order (rq.zl): the first
  // admitted one is their minimum.  Every warp runs the same scan (no
  // barrier); only the re-estimated (partially prefilled) relQueries are
  // compared by value.  Starvation overrides (finite tau) or a long run of
  // not-yet-admitted entries fall back to one block reduction over all.
  int head_l;
  int zptr_new = c.zptr;
  bool z_cache = false;  // this iteration's static-order head can be cached (thread 0, decision block)
  unsigned long long zkey = ~0ULL;
  int zidx = 0x7FFFFFFF;
  {
    const int lane = tid & 31;
    unsigned long long key = ~0ULL;
    int idx = 0x7FFFFFFF;
    const bool zorder = kC || P.zorder, use_dpu = kC || P.use_dpu;
    bool full = !zorder;
    if (zorder && c.zh_valid) {  // the static-order head is unchanged since the last scan
      key = c.zh_key;
      idx = c.zh_idx;
    } else if (zorder) {
      int i0 = c.zptr;
      bool lead = true;
      for (int round = 0;; ++round) {
        if (i0 >= T.nzl) break;
        if (round == kZScanRounds) {
          full = true;
          break;
        }
        const int i = i0 + lane;
        bool gone = true, elig = false;
        int a = 0;
        if (i < T.nzl) {
          a = rq.zl[i];
          const int q = rq.q[a], sz = rq.off[a + 1] - rq.off[a];
          // DPU policies: leaves the static order at its first prefill; sp/fcfs: when fully prefilled
          gone = use_dpu ? (q > 0 || sz == 0) : q >= sz;
          elig = !gone && a < c.n_admitted;
        }
        if (lead) {
          const unsigned keep = ~__ballot_sync(kFull, gone);
          if (keep == 0) {
            zptr_new = i0 + 32 < T.nzl ? i0 + 32 : T.nzl;
          } else {
            zptr_new = i0 + __ffs(keep) - 1;
            lead = false;
          }
        }
        const unsigned em = __ballot_sync(kFull, elig);
        if (em) {
          idx = __shfl_sync(kFull, a, __ffs(em) - 1);
          key = okey(rq.prio[idx]);
          break;
        }
        i0 += 32;
      }
    }
    zkey = key;  // the static-order head
    zidx = idx;
    z_cache = zorder && !full;
    if (zorder) {
      if (use_dpu) {  // partially prefilled relQueries with pending rows (this shard's)
        bool better = false;  // this lane holds one that beats the static-order head
        for (int j = lane; j < c.n_act; j += 32) {
          const int a = c.act[j];
          if (rq.q[a] < rq.off[a + 1] - rq.off[a] && (kC || T.shard_world == 1 || a % T.shard_world == T.shard_rank)) {
            const unsigned long long k = okey(rq.prio[a]);
            if (k < key || (k == key && a < idx)) {
              key = k;
              idx = a;
              better = true;
            }
          }
        }
        const unsigned bm = __ballot_sync(kFull, better);
        if (__popc(bm) == 1) {  // the usual case: the one relQuery being prefilled
          const int l = __ffs(bm) - 1;
          key = __shfl_sync(kFull, key, l);
          idx = __shfl_sync(kFull, idx, l);
        } else if (bm) {
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) {
            const unsigned long long ok = __shfl_xor_sync(kFull, key, d);
            const int oi = __shfl_xor_sync(kFull, idx, d);
            if (ok < key || (ok == key && oi < idx)) {
              key = ok;
              idx = oi;
            }
          }
        }
      }
    }
    if (full) {
      int w = 0;
      key = ~0ULL;
      idx = 0x7FFFFFFF;
      for (int a = tid; a < c.n_admitted; a += NT) {
        if (rq.q[a] < rq.off[a + 1] - rq.off[a] && (T.shard_world == 1 || a % T.shard_world == T.shard_rank)) {
          ++w;
          const unsigned long long k = okey(rq.prio[a]);
          if (k < key) {  // ranks visited in increasing order: strict < keeps the smallest rank
            key = k;
            idx = a;
          }
        }
      }
      group_count_argmin<GC>(w, key, idx, S.red);  // result is group-uniform in registers
    }
    if (!kC && T.shard_world > 1) {  // allgather of the shards' heads and priorities
      if (!shard_exchange(T, S, key, idx)) return false;
    }
    if (kC && T.shard_world > 1) {  // every shard has every priority: only the heads travel
      if (!shard_exchange_heads<GC>(T, S, key, idx)) {
        if constexpr (kC) {  // release group D (waiting for the candidates or the advance)
          if (tid == 0) S.go_exec = 0;
          if (!early) decision_arrive();
          exec_done_arrive();
        }
        return false;
      }
    }
    head_l = c.n_wait > 0 && idx != 0x7FFFFFFF ? idx : -1;
    if (tid == 0) {
      if (c.n_wait > 0 && head_l < 0) {  // internal inconsistency: never expected
        c.status = RS_EUNSUPPORTED;
        c.error_detail = 9;
      }
      S.W = c.n_wait;
      S.head = head_l;  // read by other threads only after later barriers
    }
  }
  // parity mode (any kernel, the common one included: the snapshot is a cold call)
  if (T.snap_prio) record_parity(P, T, S, c.n_log & (T.log_cap - 1));
  phase_mark(c, 2);

  // ---- D: candidates (engine.py:285-308)
  {
    // decode candidate = running list.  m+ = min over the distinct running
    // relQueries (rrq); the first running row attaining it only matters when
    // two distinct relQueries tie on m+.
    if (tid == 0) {
      double best = 0.0;
      int brank = -1, nties = 0;
      for (int i = 0; i < c.n_rrq; ++i) {
        const double p = rq.prio[c.rrq[i]];
        if (brank < 0 || p < best) {
          best = p;
          brank = c.rrq[i];
          nties = 1;
        } else if (p == best) {
          ++nties;
        }
      }
      if (nties > 1) {
        for (int j = 0; j < c.n_run; ++j)
          if (rq.prio[c.run_rank[j]] == best) {
            brank = c.run_rank[j];
            break;
          }
      }
      S.dmin_slot = brank;  // rank of the first running row with the minimum priority
      S.m_plus = c.n_run > 0 ? best : qnan();
      S.first_bad = 0x7FFFFFFF;
    }
    phase_mark(c, 11);
    // prefill candidate: leading run of the head's pending rows (arranger.py:80-112),
    // scanned here or -- after a decode -- already by group M while group D finished
    // the previous update (cand_scan: nothing it reads changes in between)
    const int h = head_l;
    const bool pre = kC && S.pc.valid && h >= 0 && h == S.pc.head;  // group-uniform
    int J, mh;
    if (pre) {
      J = S.pc.J;
      mh = S.pc.mh;
    } else {
      cand_scan<kC, GC>(P, T, S, h, J, mh);
    }
    if (tid == 0) {
      const int fb = pre ? S.pc.first_bad : S.first_bad;
      const int taken = fb < J ? fb : J;
      const int loaded = ((fb < J ? fb : J - 1) / NT + 1) * NT;
      c.alg_bytes += 8LL * (J < loaded ? J : loaded);  // candidate tok + out
      S.taken = taken;
      S.cand_mh = mh;
      S.utok_sum = taken > 0 ? S.cand_u[taken - 1] : 0;
      S.m_minus = taken > 0 ? rq.prio[h] : qnan();
    }
    GC::sync();
    phase_mark(c, 12);
  }
  if constexpr (kC) {
    if (!early) decision_arrive();  // the candidates: group D may start the update (see above)
  }

  // ---- E: decision (engine.py:387-433, arranger.py:115-179)
  const bool has_p = S.taken > 0, has_d = c.n_run > 0;
  const bool need_proj = (kC || !P.prefill_first) && has_p && has_d && S.dmin_slot != S.head && S.m_plus <= S.m_minus;
  if (need_proj) {
    // distinct running relQueries in rel_id order (engine.py:406-408): each one's
    // position and projection term (arranger.py:130-137), computed in parallel;
    // thread 0 then only adds the terms in order
    const int nd = c.n_rrq;
    const double adn = __dmul_rn(P.pol.alpha_d, (double)S.taken);
    const long long olp = rq.ol[S.head];
    for (int i = tid; i < nd; i += NT) {
      const int a = c.rrq[i];
      const int ri = rq.relrank[a];
      int pos = 0;
#pragma unroll 4
      for (int k = 0; k < nd; ++k) pos += rq.relrank[c.rrq[k]] < ri;
      const long long o = rq.ol[a];
      S.dterm[pos] = __dmul_rn(adn, (double)(o < olp ? o : olp));
      atomicMax(&S.max_ol, (int)o);
    }
    if (tid == 0) S.n_dist = nd;
    GC::sync();
  }
  if (tid == 0) {
    int action, kase;
    double dp, dm, dt, mp, mmn;
    arrange(P.pol, !kC && P.prefill_first, P.force, has_p, has_d, S.dmin_slot == S.head, S.m_plus, S.m_minus, S.utok_sum,
            S.taken, need_proj ? rq.ol[S.head] : 0, need_proj ? S.n_dist : 0, TermProj{S.dterm, (long long)S.max_ol},
            S.W, action, kase, mp, mmn, dp, dm, dt);
    S.max_ol = 0;  // for the next projection
    S.pc.valid = 0;  // (read by every thread of phase D before its barrier)
    S.action = action;
    c.zptr = zptr_new;
    if (z_cache) {  // valid until an admission or a prefill of that relQuery
      c.zh_key = zkey;
      c.zh_idx = zidx;
      c.zh_valid = 1;
    }
    if (kC || (cfg.log_decisions && T.log_cap > 0)) {
      c.alg_bytes += sizeof(rs_iter_record);
      rs_iter_record& r = T.log[c.n_log & (T.log_cap - 1)];
      r.iteration = c.iteration;
      r.clock = c.clock;
      r.m_plus = mp;
      r.m_minus = mmn;
      r.delta_plus = dp;
      r.delta_minus = dm;
      r.delta_total = dt;
      r.action = action;
      r.kase = kase;
      r.head = S.head;
      r.n_waiting = S.W;
      r.batch_rq = -1;
      r.batch_first = 0;
      r.batch_n = 0;
      r.n_reestimated = S.n_est;
      r.kv_reserved = 0;
    }
  }
  GC::sync();
  const int action = S.action;
  phase_mark(c, 3);

  // ---- F: execute
  if constexpr (kC) {
    // pipelined: group M executes this iteration while group D computes the
    // next iteration's priority update of the partially prefilled relQueries
    // (dpu_spec, started after phase B) from the state this advance leaves.
    // The groups do not join here: group M signals the advance done (barrier
    // kBarExecDone, arrive only) and goes on to the next iteration's admission;
    // group D, once its update is computed, waits for that signal, commits the
    // update against the advance's result, and both meet at the admission
    // barrier -- so the update may run over into the admission.
    const bool go = execute<kC, GM, true>(P, T, S, action);  // group-uniform
    if (tid == 0) S.go_exec = go;
    exec_done_arrive();
    if (go && action == RS_ACTION_DECODE && S.head >= 0) {
      // a decode leaves the waiting queue, the head's rows and chain as they were and
      // group D's update is the longer branch: scan the next prefill candidate now,
      // for the (likely unchanged) head (used by phase D if it is still the head)
      const int hp = S.head;
      if (tid == 0) S.first_bad = 0x7FFFFFFF;
      GM::sync();
      int J, mh;
      cand_scan<kC, GM>(P, T, S, hp, J, mh);
      if (tid == 0) {
        S.pc.head = hp;
        S.pc.J = J;
        S.pc.mh = mh;
        S.pc.first_bad = S.first_bad;
        S.pc.valid = 1;
      }
    }
    return go;
  } else {
    return execute<kC, GAll, false>(P, T, S, action);
  }
}

__device__ __forceinline__ void copy16(void* dst, const void* src, size_t bytes) {
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  for (size_t i = threadIdx.x; i < bytes / 16; i += kThreads) d[i] = s[i];
}

// kPart (common configuration, a relQuery table in HBM: configs 3 and 5): the
// pipelined update may cover the first kSmallEst entries of a longer list
template <bool kFast, bool kC, bool kPart = false>
__global__ void __launch_bounds__(kThreads, 1) engine_kernel(Params P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ TraceDev Tsm;  // the trace's pointers, read on every access
  Shared& S = *reinterpret_cast<Shared*>(smem_raw);

  if (threadIdx.x == 0) Tsm = P.traces[blockIdx.x];
  __syncthreads();
  const TraceDev& T = Tsm;
  copy16(&S.c, T.ctl, sizeof(Ctl));
  for (int i = threadIdx.x; i < kJumpBits; i += kThreads) S.jt[i] = T.jump[i];
  for (int i = threadIdx.x; i < 32; i += kThreads) S.jstep[i] = T.jump[kJumpBits + i];
  const size_t rqb = rq_bytes(T.R);
  void* rq_base = T.rq_in_smem ? (void*)(smem_raw + ((sizeof(Shared) + 15) & ~(size_t)15)) : T.rq_global;
  if (T.rq_in_smem) copy16(rq_base, T.rq_global, rqb);
  if (threadIdx.x == 0) {
    S.rq = rq_carve(rq_base, T.R);
    S.pf_head = -1;  // no previous head to prefetch for
    S.spec_ok = 0;   // the launch's first update runs in place (dpu_update)
    S.max_ol = 0;
    S.pc.valid = 0;
  }
  __syncthreads();
  if (S.c.status == RS_RUNNING) {
    if (threadIdx.x == 0) S.c.phase[kPhases - 1] = clock64();
    for (long long it = 0; it < P.max_iters; ++it)
      if (!iterate<kFast, kC, kPart>(P, T, S, it + 1 == P.max_iters)) break;
  }
  __syncthreads();
  // running rows' generated counts back to HBM (finished rows were written at completion)
  for (int j = threadIdx.x; j < S.c.n_run; j += kThreads) T.gen[S.c.run_row[j]] = S.c.run_gen[j];
  if (T.rq_in_smem) copy16(T.rq_global, rq_base, rqb);
  copy16(T.ctl, &S.c, sizeof(Ctl));
}

// ---------------------------------------------------------------------------
// Unit kernels
// ---------------------------------------------------------------------------

struct ArrItems {
  const long long* utok;
  const int* rem;
  const unsigned char* pre;
  long long off;
  __device__ __forceinline__ void item(int t, long long& u, int& r, int& p) const {
    u = utok[off + t];
    r = rem[off + t];
    p = pre[off + t];
  }
};

struct ArrSetItems {  // one set as a batch of one
  const long long* utok;
  const int* rem;
  const unsigned char* pre;
  long long off;
  int n;
  __device__ __forceinline__ int count(int) const { return n; }
  __device__ __forceinline__ void item(int, int i, long long& u, int& r, int& p) const {
    u = utok[off + i];
    r = rem[off + i];
    p = pre[off + i];
  }
};

struct ValOut {
  double* out;
  long long s;
  __device__ __forceinline__ void operator()(int, double v) const { out[s] = v; }
};

struct UnitShared {
  SegShared sh;
  PrefixSummary ps[1];
  long long U[kItemBuf];
  double terms[2 * kItemBuf + kEstBatch];
  int UNP[kItemBuf];
  int REM[kItemBuf];
  int jcnt[kItemBuf + kEstBatch];
  int io[2];
  int jo[2];
};

// one CTA per remainder: the engine's segment-parallel PEM when mns*max(utok)
// <= cap (seg_ok[s]) and the remainder fits the staging buffers, else the
// engine's warp PEM
__global__ void __launch_bounds__(kThreads)
    pem_batch_kernel(long long n_sets, const long long* item_off, const long long* utok, const int* rem,
                     const unsigned char* pre, const unsigned char* seg_ok, PemModel m, double* out) {
  extern __shared__ __align__(16) unsigned char unit_smem[];
  UnitShared& S = *reinterpret_cast<UnitShared*>(unit_smem);
  for (long long s = blockIdx.x; s < n_sets; s += gridDim.x) {
    const int n = (int)(item_off[s + 1] - item_off[s]);
    if (seg_ok[s] && n <= kItemBuf) {
      if (threadIdx.x == 0) S.ps[0] = PrefixSummary{0, 0, 0};
      __syncthreads();
      SegBuf sb{S.U, S.UNP, S.REM, S.terms, S.jcnt, S.io, S.jo};
      seg_pem_batch(ArrSetItems{utok, rem, pre, item_off[s], n}, 1, S.ps, m, sb, S.sh, ValOut{out, s});
    } else if (threadIdx.x < 32) {
      ArrItems it{utok, rem, pre, item_off[s]};
      const PrefixSummary none{0, 0, 0};
      const double v = warp_pem(it, n, none, m);
      if (threadIdx.x == 0) out[s] = v;
    }
    __syncthreads();
  }
}

__global__ void choice_kernel(rs_pcg64_state* st, long long n_calls, const long long* n, const long long* k,
                              long long* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Pcg64 g = Pcg64::from(*st);
  long long o = 0;
  for (long long c = 0; c < n_calls; ++c) {
    uint32_t idx[kMaxSample];
    choice_floyd(g, (uint32_t)n[c], (uint32_t)k[c], idx);
    for (long long i = 0; i < k[c]; ++i) out[o + i] = idx[i];
    o += k[c];
  }
  *st = g.to();
}

// Unit entry point of the arranger (rs_arrange): rank the distinct running
// relQueries by rel_id as the engine does (engine.py:406-408), then thread 0
// runs the engine's arrange().
__global__ void arrange_kernel(int n_run, const long long* run_rel, const long long* run_ol, long long d_min_rel,
                               int n_p, long long utok_sum, long long p_rel, long long ol_p, double m_plus,
                               double m_minus, long long W, int prefill_first, int force, rs_cost_model m,
                               long long* sorted_ol, rs_iter_record* out) {
  for (int i = threadIdx.x; i < n_run; i += blockDim.x) {
    int pos = 0;
    for (int k = 0; k < n_run; ++k) pos += run_rel[k] < run_rel[i];
    sorted_ol[pos] = run_ol[i];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int action, kase;
  double mp, mmn, dp, dm, dt;
  arrange(m, prefill_first, force, n_p > 0, n_run > 0, n_run > 0 && n_p > 0 && d_min_rel == p_rel, m_plus, m_minus,
          utok_sum, n_p, ol_p, n_run, OlProj{sorted_ol}, W, action, kase, mp, mmn, dp, dm, dt);
  rs_iter_record r{};
  r.m_plus = mp;
  r.m_minus = mmn;
  r.delta_plus = dp;
  r.delta_minus = dm;
  r.delta_total = dt;
  r.action = action;
  r.kase = kase;
  r.n_waiting = (int)W;
  r.batch_n = n_p;
  *out = r;
}

// First-sight priorities of every relQuery (one warp each, whole grid): PEM
// of all rows with utok = tok, remaining = output_limit (see first_sight()).
struct StaticItems {
  const int* tok;
  int base, ol;
  __device__ __forceinline__ void item(int t, long long& u, int& rem, int& pre) const {
    u = tok[base + t];
    rem = ol;
    pre = 0;
  }
};

__global__ void __launch_bounds__(kThreads) first_sight_kernel(int R, const int* off, const int* ol, const int* tok,
                                                               PemModel m, double* out) {
  const int warps = gridDim.x * kWarps;
  for (int a = blockIdx.x * kWarps + (threadIdx.x >> 5); a < R; a += warps) {
    const PrefixSummary none{0, 0, 0};
    const double v = warp_pem(StaticItems{tok, off[a], ol[a]}, off[a + 1] - off[a], none, m);
    if ((threadIdx.x & 31) == 0) out[a] = v;
  }
}

// First sight, segment-parallel (when PEM segments close by count only,
// mns <= 256): a whole-grid, bandwidth-shaped pass that reads each row's tok
// once.  One THREAD per PEM segment of every relQuery walks the segment's rows
// in order -- pem()'s own scan (priority.py:187-217) with every row unprefilled,
// utok = tok and remaining = output_limit: a prefill sub-batch closes before a
// row that would take it past mnbt -- and writes the segment's terms in the
// reference's order (its sub-batches, then the decode term);
// first_sight_sum_kernel then adds each relQuery's terms in order.  A warp thus
// advances 32 segments at once with a handful of instructions per row, instead
// of one segment's sequential sub-batch chain per warp; each lane reads its rows
// by whole cache lines, two lines in flight, so HBM sees every line once.
// seg[sg] = (first row, rows, output limit) of segment sg (host-built).
// Terms per segment are bounded by 2*sum(tok)/mnbt + 3 (consecutive next-fit
// sub-batches exceed mnbt together); the host sizes `bound` from max(tok).
// One 32-row line of a segment's scan: rows outside [vlo, vhi) of the line are
// another segment's and are skipped (kMask: the line may hold such rows).
template <bool kMask>
__device__ __forceinline__ void fs_scan_line(const int4 (&q)[8], int vlo, int vhi, int mnbt, int& p, int& nt,
                                             double* tj, const PemModel& m) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int4 v = q[i >> 2];
    int u = (i & 3) == 0 ? v.x : (i & 3) == 1 ? v.y : (i & 3) == 2 ? v.z : v.w;
    if (kMask) u = (i >= vlo && i < vhi) ? u : 0;
    const int np = p + u;  // every row has tok >= 1: p > 0 <=> the sub-batch is non-empty
    if (np > mnbt && p > 0 && u > 0) {  // the row would take the sub-batch past mnbt (priority.py:205-208)
      tj[nt++] = lin(m.ap, (double)p, m.bp);
      p = u;
    } else {
      p = np;
    }
  }
}

__global__ void __launch_bounds__(256) first_sight_seg_kernel(int n_seg, const int4* seg, const int* tok, PemModel m,
                                                              int bound, double* terms, int* nterm) {
  const int mnbt = (int)m.mnbt;
  for (int sg = blockIdx.x * blockDim.x + threadIdx.x; sg < n_seg; sg += gridDim.x * blockDim.x) {
    const int4 d = seg[sg];
    // rows [d.x, d.x + d.y) read by whole 128-byte lines (8 x 16 B in flight, the
    // next line prefetched while this one is scanned); only the first and last
    // lines can hold other segments' rows
    const int lo = d.x & ~31, hi = d.x + d.y;
    const int4* t4 = reinterpret_cast<const int4*>(tok + lo);
    double* tj = terms + (size_t)sg * bound;
    int nt = 0, p = 0;  // p = p_utok of pem()
    int4 cur[8], nxt[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) cur[i] = lo + 4 * i < hi ? __ldg(t4 + i) : make_int4(0, 0, 0, 0);
    for (int r0 = lo; r0 < hi; r0 += 32) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        nxt[i] = r0 + 32 + 4 * i < hi ? __ldg(t4 + ((r0 + 32 - lo) >> 2) + i) : make_int4(0, 0, 0, 0);
      if (r0 >= d.x && r0 + 32 <= hi) fs_scan_line<false>(cur, 0, 32, mnbt, p, nt, tj, m);
      else fs_scan_line<true>(cur, d.x - r0, hi - r0, mnbt, p, nt, tj, m);
#pragma unroll
      for (int i = 0; i < 8; ++i) cur[i] = nxt[i];
    }
    if (p > 0) tj[nt++] = lin(m.ap, (double)p, m.bp);
    const long long o = d.z;
    tj[nt] = __dadd_rn(__dmul_rn(m.ad, (double)((long long)d.y * o)), __dmul_rn(m.bd, (double)o));
    nterm[sg] = nt + 1;
  }
}

__global__ void first_sight_sum_kernel(int R, const int* seg_pref, int bound, const double* terms, const int* nterm,
                                       double* out) {
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < R; a += gridDim.x * blockDim.x) {
    double total = 0.0;  // pem() accumulates its terms in scan order (priority.py:197-218)
    for (int sg = seg_pref[a]; sg < seg_pref[a + 1]; ++sg) {
      const double* tj = terms + (size_t)sg * bound;
      const int nt = nterm[sg];
      for (int i = 0; i < nt; ++i) total = __dadd_rn(total, tj[i]);
    }
    out[a] = total;
  }
}

// Engine-creation row checks (engine.py:235-239 and the device model's limits),
// one warp per relQuery over the uploaded rows: res[0] = the first admission
// rank with an offending row (INT_MAX if none), res[1] = the largest tok.  The
// host names the offending row only when res[0] says there is one.
__global__ void __launch_bounds__(kThreads) validate_rows_kernel(int R, const int* off, const int* ol, const int* chain,
                                                                 const int* tok, const int* out, long long B,
                                                                 long long cap, int* res) {
  const int warps = gridDim.x * kWarps, lane = threadIdx.x & 31;
  for (int a = blockIdx.x * kWarps + (threadIdx.x >> 5); a < R; a += warps) {
    const int lo = off[a], hi = off[a + 1];
    if (hi == lo) continue;
    int tmin = 0x7FFFFFFF, tmax = -0x7FFFFFFF - 1, omin = 0x7FFFFFFF, omax = -0x7FFFFFFF - 1;
    for (int i = lo + lane; i < hi; i += 32) {
      const int t = tok[i], o = out[i];
      tmin = t < tmin ? t : tmin;
      tmax = t > tmax ? t : tmax;
      omin = o < omin ? o : omin;
      omax = o > omax ? o : omax;
    }
    tmin = __reduce_min_sync(kFull, tmin);
    tmax = __reduce_max_sync(kFull, tmax);
    omin = __reduce_min_sync(kFull, omin);
    omax = __reduce_max_sync(kFull, omax);
    if (lane == 0) {
      const long long o = ol[a];
      if (tmin <= 0 || omin < 1 || omax > o || tmax + o > cap || tmax + o >= (1LL << 20) ||
          tmin < (long long)chain[a] * B)
        atomicMin(&res[0], a);
      atomicMax(&res[1], tmax);
    }
  }
}

// Unit entry point of the waiting order (rs_waiting_argmin): the engine's
// full-scan head reduction -- ranks visited in increasing order with a strict
// `<`, then block_count_argmin -- over given priorities and waiting flags.
__global__ void __launch_bounds__(kThreads) waiting_argmin_kernel(long long n, const double* prio,
                                                                  const unsigned char* waiting, long long* out) {
  __shared__ RedSmem red;
  int w = 0;
  unsigned long long key = ~0ULL;
  int idx = 0x7FFFFFFF;
  for (long long a = threadIdx.x; a < n; a += kThreads) {
    if (waiting[a]) {
      ++w;
      const unsigned long long k = okey(prio[a]);
      if (k < key) {
        key = k;
        idx = (int)a;
      }
    }
  }
  block_count_argmin(w, key, idx, red);
  if (threadIdx.x == 0) {
    out[0] = idx == 0x7FFFFFFF ? -1 : idx;
    out[1] = w;
  }
}

}  // namespace rsd

// ===========================================================================
// Host side: C ABI
// ===========================================================================

using namespace rsd;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// RS_TIMING=1 in the environment: host-side phase times of engine creation on stderr
struct PhaseClock {
  bool on = getenv("RS_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[rs] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

#define RS_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess) return fail(RS_ECUDA, std::string(#call ": ") + cudaGetErrorString(_e)); \
  } while (0)

// A host column shared (not copied) between the replicas of a sharded pool;
// copy-on-write for the rare replica that changes one.
template <class T>
struct SharedVec {
  std::shared_ptr<std::vector<T>> p = std::make_shared<std::vector<T>>();
  std::vector<T>& w() {
    if (p.use_count() > 1) p = std::make_shared<std::vector<T>>(*p);
    return *p;
  }
  const T& operator[](size_t i) const { return (*p)[i]; }
  T& operator[](size_t i) { return w()[i]; }
  size_t size() const { return p->size(); }
  bool empty() const { return p->empty(); }
  const T* cdata() const { return p->data(); }
  T* data() { return w().data(); }
  typename std::vector<T>::iterator begin() { return w().begin(); }
  typename std::vector<T>::iterator end() { return w().end(); }
  void resize(size_t n) { w().resize(n); }
  void assign(size_t n, const T& v) { w().assign(n, v); }
  template <class It>
  void assign(It a, It b) { w().assign(a, b); }
};

struct HostTrace {
  TraceDev dev{};
  rs_cost_model pol{};
  SharedVec<unsigned char> rq_host;  // relQuery table staging (rq_carve layout)
  SharedVec<int> off;                // rank-ordered row offsets
  SharedVec<int> rank_of;     // trace index -> rank
  SharedVec<int> order;       // rank -> trace index
  SharedVec<long long> row_src;  // rank-ordered row -> trace-order row (empty: identity)
  std::vector<void*> allocs;
  long long bytes = 0;
  long long log_read = 0;
  // one device arena per trace (a cudaMalloc per buffer costs more than the upload itself)
  char* arena = nullptr;
  void* arena_alloc = nullptr;  // cudaMallocAsync (pool) allocation
  size_t arena_cap = 0, arena_used = 0;
  size_t arena_top = 0;  // staging: buffers needing no initialisation are carved from the top (never uploaded)
  double* noise_buf = nullptr;  // rs_engine_set_noise
  // small traces: arena contents are composed in a host image and uploaded in
  // one copy per flush (stage_flush) instead of a copy / memset per buffer
  bool staging = false;
  std::vector<unsigned char> stage;
  size_t staged_lo = 0;  // arena bytes [staged_lo, arena_used) not uploaded yet
  SharedVec<int> zorder;      // every relQuery in the static waiting order
  bool no_log = false;          // created with log_capacity 0 (the device writes a scratch record)
  // small traces: the staged arena image and the creation kernels wait for one
  // engine-wide upload (finish_deferred)
  bool deferred = false;
  std::vector<std::function<int()>> pending;  // kernel launches after the upload, in order
};

// Page-locked staging for the deferred uploads of engine creation, reused
// across engines (allocating page-locked memory costs far more than the copy);
// a reuse waits for the previous creation's copies (an event).
struct PinnedStage {
  std::mutex mu;
  unsigned char* p = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
};
PinnedStage g_pinned;

// Reserve the trace's arena: every dalloc below carves from it (256-byte aligned).
// The arena comes from the device's stream-ordered pool, which keeps freed
// memory (release threshold = max): re-creating an engine of the same shape
// reuses it instead of mapping fresh pages (a cudaMalloc/cudaFree round trip
// of tens of MB costs milliseconds).
void keep_pool(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[device] = true;
}

int arena_reserve(HostTrace& h, size_t bytes) {
  void* q = nullptr;
  bytes = (bytes + 255) & ~(size_t)255;  // both ends of the arena carve 256-byte aligned buffers
  cudaError_t e = cudaMallocAsync(&q, bytes, 0);
  if (e != cudaSuccess) return fail(RS_ENOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
  h.arena_alloc = q;
  h.arena = (char*)q;
  h.arena_cap = bytes;
  h.arena_top = bytes;
  h.arena_used = 0;
  return RS_OK;
}

int stage_flush(HostTrace& h) {  // upload the staged arena bytes composed since the last flush
  if (!h.staging || h.arena_used <= h.staged_lo) return RS_OK;
  const cudaError_t e = cudaMemcpy(h.arena + h.staged_lo, h.stage.data() + h.staged_lo, h.arena_used - h.staged_lo,
                                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fail(RS_ECUDA, std::string("staged upload: ") + cudaGetErrorString(e));
  h.staged_lo = h.arena_used;
  return RS_OK;
}

template <typename T>
int dalloc(HostTrace& h, T** p, size_t n, const void* src = nullptr, int fill_byte = -1, bool async = false) {
  if (n == 0) n = 1;
  void* q = nullptr;
  const size_t nb = (n * sizeof(T) + 255) & ~(size_t)255;
  if (h.staging && h.arena && !src && fill_byte < 0 && h.arena_used + nb <= h.arena_top) {
    // no contents: from the top of the arena, outside the uploaded image
    h.arena_top -= nb;
    h.bytes += (long long)(n * sizeof(T));
    *p = (T*)(h.arena + h.arena_top);
    return RS_OK;
  }
  if (h.staging && !h.deferred && h.arena && h.arena_used + nb <= h.arena_top && !src && fill_byte >= 0 &&
      nb >= (64u << 10)) {
    // a large fill (the decision-log ring): flush what is composed, fill on the device
    int rc = stage_flush(h);
    if (rc) return rc;
    q = h.arena + h.arena_used;
    h.arena_used += nb;
    h.staged_lo = h.arena_used;
    h.bytes += (long long)(n * sizeof(T));
    const cudaError_t e = cudaMemsetAsync(q, fill_byte, n * sizeof(T), 0);
    if (e != cudaSuccess) return fail(RS_ECUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
    *p = (T*)q;
    return RS_OK;
  }
  if (h.staging && h.arena && h.arena_used + nb <= h.arena_top) {  // composed on the host
    const size_t at = h.arena_used;
    h.arena_used += nb;
    h.bytes += (long long)(n * sizeof(T));
    h.stage.resize(h.arena_used);  // grows with the image (capacity reserved up front)
    if (src) memcpy(h.stage.data() + at, src, n * sizeof(T));
    else if (fill_byte >= 0) memset(h.stage.data() + at, fill_byte, n * sizeof(T));
    *p = (T*)(h.arena + at);
    return RS_OK;
  }
  if (h.arena && h.arena_used + nb <= h.arena_top) {
    q = h.arena + h.arena_used;
    h.arena_used += nb;
  } else {
    cudaError_t e = cudaMalloc(&q, n * sizeof(T));
    if (e != cudaSuccess) return fail(RS_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    h.allocs.push_back(q);
  }
  h.bytes += (long long)(n * sizeof(T));
  cudaError_t e = cudaSuccess;
  if (src) {
    e = async ? cudaMemcpyAsync(q, src, n * sizeof(T), cudaMemcpyHostToDevice, 0)
              : cudaMemcpy(q, src, n * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(RS_ECUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
  } else if (fill_byte >= 0) {
    e = cudaMemset(q, fill_byte, n * sizeof(T));
    if (e != cudaSuccess) return fail(RS_ECUDA, std::string("cudaMemset: ") + cudaGetErrorString(e));
  }
  *p = (T*)q;
  return RS_OK;
}

struct DevBuf {  // scratch freed on every return path
  std::vector<void*> p;
  template <typename T>
  cudaError_t get(T** out, size_t n) {
    void* q = nullptr;
    const cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) p.push_back(q);
    *out = (T*)q;
    return e;
  }
  ~DevBuf() {
    for (void* q : p) cudaFree(q);
  }
};

// keys of the static waiting order: okey(priority) per rank, values = the ranks
__global__ void static_keys_kernel(const double* prio, int R, unsigned long long* key, int* val) {
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < R; a += gridDim.x * blockDim.x) {
    key[a] = okey(prio[a]);
    val[a] = a;
  }
}

}  // namespace

// Stable sort of n (key, value) device pairs by key in place (radix_sort.cuh):
// one CTA up to kSortOneCta pairs, else the multi-CTA passes.
static int sort_pairs_dev(unsigned long long* k, int* v, long long n, cudaStream_t st) {
  if (n <= 1) return RS_OK;
  DevBuf b;
  unsigned long long* k1 = nullptr;
  int* v1 = nullptr;
  RS_CUDA(b.get(&k1, n));
  RS_CUDA(b.get(&v1, n));
  if (n <= kSortOneCta) {
    sort_pairs_one_cta<<<1, kSortThreads, 0, st>>>(k, v, k1, v1, (int)n);
    RS_CUDA(cudaGetLastError());
    RS_CUDA(cudaStreamSynchronize(st));  // the scratch is freed on return
    return RS_OK;
  }
  const long long tiles = (n + kSortTile - 1) / kSortTile;
  unsigned long long* gh = nullptr;
  unsigned* th = nullptr;
  RS_CUDA(b.get(&gh, 8 * 256));
  RS_CUDA(b.get(&th, 256 * tiles));
  RS_CUDA(sort_pairs_enqueue(k, v, k1, v1, gh, th, n, st));
  RS_CUDA(cudaStreamSynchronize(st));
  return RS_OK;
}


struct rs_engine {
  int device = 0;
  int shard_world = 1, shard_rank = 0;  // sharded pool (rs_engine_create_sharded); rank -1: all shards here
  ShardRec* mbox = nullptr;              // this engine's mailbox(es)
  ShardRec** d_peers = nullptr;          // device array [world] of peer mailbox pointers
  bool mbox_pooled = false;              // mailboxes from the stream-ordered pool (all shards in this process)
  bool connected = true;                 // one-shard engines: peers' mailboxes known (rs_engine_connect)
  bool fast = true;  // every trace qualifies for engine_kernel<true, *>
  bool common = false;  // ... and the configuration is the common one (engine_kernel<true, true>)
  bool part = false;    // ... with a relQuery table in HBM (engine_kernel<true, true, true>)
  Params params{};
  std::vector<HostTrace> traces;
  TraceDev* d_traces = nullptr;
  size_t smem = 0;
  cudaEvent_t done = nullptr;  // recorded after every launch: destroy waits on it before the stream-ordered frees
  cudaEvent_t ready = nullptr;  // creation's asynchronous uploads and kernels (legacy stream) are complete
};

extern "C" {

const char* rs_last_error(void) { return g_err.c_str(); }

const char* rs_build_info(void) {
  return "relserve-b200: sm_100a persistent scheduler CTA (" __DATE__ ")";
}

static int validate_config(const rs_config* cfg) {
  if (cfg->policy < RS_POLICY_FCFS || cfg->policy > RS_POLICY_RELSERVE_DP)
    return fail(RS_EINVAL, "unknown policy");
  if (cfg->cap <= 0 || cfg->max_num_seqs <= 0 || cfg->max_num_batched_tokens <= 0)
    return fail(RS_EINVAL, "constraints must be positive");
  if (cfg->max_num_batched_tokens > cfg->cap)
    return fail(RS_EINVAL, "max_num_batched_tokens must not exceed cap");
  if (cfg->block_size <= 0 || cfg->capacity_blocks <= 0)
    return fail(RS_EINVAL, "block_size and capacity_blocks must be positive");
  const bool dpu = cfg->policy >= RS_POLICY_RELSERVE;
  if (dpu && !(cfg->tau > 0)) return fail(RS_EINVAL, "tau must be positive");
  if (!(cfg->noise_sigma >= 0)) return fail(RS_EINVAL, "noise_sigma must be non-negative");
  if (dpu && cfg->sample_size < 1) return fail(RS_EINVAL, "sample_size must be positive");
  if (dpu && cfg->sample_size > kMaxSample)
    return fail(RS_EUNSUPPORTED, "sample_size above the device limit (64)");
  if (cfg->max_num_seqs > kMaxRun) return fail(RS_EUNSUPPORTED, "max_num_seqs above the device limit (1024)");
  return RS_OK;
}

// Upper bound of one trace's arena (build_trace's buffers, 256-byte aligned each).
static size_t arena_need(const rs_trace_view& v, const rs_config* cfg, long long log_cap) {
  const size_t R = (size_t)std::max<long long>(v.num_relqueries, 0), N = (size_t)std::max<long long>(v.num_requests, 0);
  long long fifo_cap = 1;
  while (fifo_cap < cfg->capacity_blocks + kMaxRun + 2) fifo_cap <<= 1;
  long long lc = 1;  // a one-record ring when no log is kept
  while (lc < log_cap) lc <<= 1;
  const size_t need = 16 * N + 24 * R + 8 * (size_t)kMaxJobs * (kSmallMns + 1) + 8 * (R + 1) + 8 * R + 8 * (R + 1) +
                      4 * R + rq_bytes((int)R) + 16 + (size_t)fifo_cap * sizeof(FifoEnt) +
                      (kJumpBits + 32) * sizeof(JumpEntry) + (size_t)lc * sizeof(rs_iter_record) + sizeof(Ctl) +
                      12 * (R + 1) + 8 + 24 * R /* static-order sort scratch */ +
                      8 * 8 * 256 + 4 * 256 * (R / kSortTile + 1) /* ... its grid passes' histograms */ +
                      4 * (R + 1) /* first-sight segments */ +
                      16 * (R + N / (size_t)std::max<long long>(cfg->max_num_seqs, 1) + 1) /* ... their descriptors */ +
                      47 * 256;
  return (need + 255) & ~(size_t)255;
}

static int build_trace(const rs_trace_view& v, const rs_config* cfg, const rs_cost_model& pol,
                       const rs_pcg64_state& rng, long long log_cap, HostTrace& h, int shard_world = 1,
                       int shard_rank = 0) {
  h.pol = pol;
  PhaseClock pc;
  const long long R = v.num_relqueries, N = v.num_requests;
  if (R < 0 || N < 0 || R > 0x7FFFFFF0LL || N > 0x7FFFFFF0LL) return fail(RS_EINVAL, "trace too large");
  if (v.row_off[0] != 0 || v.row_off[R] != N) return fail(RS_EINVAL, "row_off must span [0, N]");
  const bool dpu = cfg->policy >= RS_POLICY_RELSERVE;
  if (cfg->policy == RS_POLICY_SP && !v.static_prio) return fail(RS_EINVAL, "sp policy needs static_prio");
  // admission order: sorted by (arrival, rel_id) (engine.py:211-213)
  h.order.resize(R);
  std::iota(h.order.begin(), h.order.end(), 0);
  std::stable_sort(h.order.begin(), h.order.end(), [&](int a, int b) {
    if (v.arrival[a] != v.arrival[b]) return v.arrival[a] < v.arrival[b];
    return v.rel_id[a] < v.rel_id[b];
  });
  h.rank_of.resize(R);
  for (long long r = 0; r < R; ++r) h.rank_of[h.order[r]] = (int)r;
  std::vector<double> arrival(R), sprio(R, 0.0);
  std::vector<int> off(R + 1), ol(R), chain(R);
  std::vector<long long> relid(R);
  // admission order == trace order (the common case: entries sorted by
  // arrival, then rel_id): rows are uploaded straight from the caller's arrays
  bool ident = true;
  for (long long a = 0; a < R && ident; ++a) ident = h.order[a] == a;
  std::vector<int> tok_buf(ident ? 0 : N), out_buf(ident ? 0 : N);
  int* tok = ident ? const_cast<int*>(v.tok) : tok_buf.data();
  int* out = ident ? const_cast<int*>(v.out) : out_buf.data();
  if (!ident) h.row_src.resize(N);
  int max_size = 1;
  long long max_nb = 0, max_tok_all = 0;
  off[0] = 0;
  for (long long a = 0; a < R; ++a) {  // per-relQuery columns in admission order (O(R))
    const int t = h.order[a];
    arrival[a] = v.arrival[t];
    ol[a] = v.output_limit[t];
    chain[a] = v.chain_blocks ? v.chain_blocks[t] : 0;
    relid[a] = v.rel_id[t];
    if (v.static_prio) {  // any number: the waiting order compares okey() keys; -0.0 ties with 0.0 there
      const double p = v.static_prio[t];
      if (p != p) return fail(RS_EINVAL, "static priority is NaN");
      sprio[a] = p == 0.0 ? 0.0 : p;
    }
    const long long lo = v.row_off[t], hi = v.row_off[t + 1];
    if (hi < lo) return fail(RS_EINVAL, "row_off must be non-decreasing");
    if (ol[a] <= 0) return fail(RS_EINVAL, "output_limit must be positive");
    if (hi - lo > max_size) max_size = (int)(hi - lo);
    if (dpu && cfg->sample_size > 200 && hi - lo > 10000)
      return fail(RS_EUNSUPPORTED, "Generator.choice tail-shuffle branch is not replayed");
    off[a + 1] = off[a] + (int)(hi - lo);
  }
  int rc;
#define TRY(x) \
  if ((rc = (x))) return rc
  {  // arena: an upper bound of every buffer below (+256 B alignment slack each)
    const size_t need = arena_need(v, cfg, log_cap);
    if (h.arena_cap >= need) {  // a slice of the engine-wide arena (create_impl)
      h.arena_top = h.arena_cap;
      h.arena_used = 0;
    } else {
      TRY(arena_reserve(h, need));
    }
    if (N < (1LL << 16)) {  // small trace: compose the arena on the host, upload it with the others at the end
      h.staging = true;
      h.deferred = shard_world == 1;
      h.stage.clear();
      h.stage.reserve(need);
      h.staged_lo = 0;
    }
  }
  // admission order == trace order: the caller's rows go up now (stream 0, asynchronous
  // from page-locked memory) while the host threads below validate them
  struct Drain {
    bool on = false;
    ~Drain() {
      if (on) cudaStreamSynchronize(0);  // the caller's buffers outlive the copy on every return path
    }
  } drain;
  TraceDev& d = h.dev;
  if (ident) {
    drain.on = true;
    TRY(dalloc(h, (int**)&d.tok, N, tok, -1, true));
    TRY(dalloc(h, (int**)&d.out, N, out, -1, true));
  }
  // rows (O(N), the bulk of creation at 10^6-10^7 rows): gather into admission
  // order unless it is the trace order, and per-relQuery min / max of tok and
  // out, on host threads over contiguous row ranges
  std::vector<int> st;  // tmin, tmax, omin, omax per relQuery
  auto scan_rows = [&](long long a0, long long a1) {
    for (long long a = a0; a < a1; ++a) {
      const long long k = off[a], n = off[a + 1] - off[a];
      if (n == 0) continue;
      if (!ident) {
        const long long lo = v.row_off[h.order[a]];
        memcpy(&tok[k], v.tok + lo, n * sizeof(int));
        memcpy(&out[k], v.out + lo, n * sizeof(int));
        std::iota(h.row_src.begin() + k, h.row_src.begin() + k + n, lo);
      }
      int tmin = tok[k], tmax = tok[k], omin = out[k], omax = out[k];
      for (long long i = k; i < k + n; ++i) {
        tmin = std::min(tmin, tok[i]);
        tmax = std::max(tmax, tok[i]);
        omin = std::min(omin, out[i]);
        omax = std::max(omax, out[i]);
      }
      st[4 * a] = tmin, st[4 * a + 1] = tmax, st[4 * a + 2] = omin, st[4 * a + 3] = omax;
    }
  };
  auto host_scan = [&]() {
    st.assign(4 * R, 0);
    const unsigned hw = std::thread::hardware_concurrency();
    const int nth = (int)std::max<long long>(1, std::min<long long>({N >> 17, 16, hw ? (long long)hw : 1}));
    std::vector<std::thread> pool;
    long long a0 = 0;
    for (int w = 0; w < nth; ++w) {  // split by rows: thread w takes relQueries up to row N*(w+1)/nth
      const long long row_end = N * (w + 1) / nth;
      long long a1 = a0;
      while (a1 < R && (w == nth - 1 || off[a1] < row_end)) ++a1;
      if (w == nth - 1) a1 = R;
      if (a1 > a0) {
        bool spawned = false;
        if (w < nth - 1) {
          try {  // no exception may cross the C ABI: a thread that cannot start scans inline
            pool.emplace_back(scan_rows, a0, a1);
            spawned = true;
          } catch (...) {
          }
        }
        if (!spawned) scan_rows(a0, a1);
      }
      a0 = a1;
    }
    for (auto& th : pool) th.join();
  };
  auto check_rows = [&]() -> int {
    for (long long a = 0; a < R; ++a) {  // checks (engine.py:235-239), in admission order
      if (off[a + 1] == off[a]) continue;
      const int tmin = st[4 * a], tmax = st[4 * a + 1], omin = st[4 * a + 2], omax = st[4 * a + 3];
      const long long lim_lo = (long long)chain[a] * cfg->block_size;  // nb >= chain  <=>  tok >= chain * B
      if (tmin <= 0 || omin < 1 || omax > ol[a] || (long long)tmax + ol[a] > cfg->cap ||
          (long long)tmax + ol[a] >= (1LL << 20) || tmin < lim_lo) {
        const long long lo = v.row_off[h.order[a]], hi = v.row_off[h.order[a] + 1];
        for (long long r = lo; r < hi; ++r) {  // name the offending row
          const long long tk = v.tok[r], ou = v.out[r];
          if (tk <= 0) return fail(RS_EINVAL, "request tokens must be non-empty");
          if (ou < 1 || ou > ol[a]) return fail(RS_EINVAL, "actual_output_len out of range");
          if (tk + ol[a] > cfg->cap) {
            char msg[200];
            snprintf(msg, sizeof msg, "request %lld/%lld needs %lld KV tokens > cap %lld", (long long)relid[a],
                     (long long)(r - lo), tk + ol[a], (long long)cfg->cap);
            return fail(RS_EINFEASIBLE, msg);
          }
          if (tk + ol[a] >= (1LL << 20))
            return fail(RS_EUNSUPPORTED, "tok + output_limit must be below 2^20 (32-bit device prefix sums)");
          if (tk < lim_lo) return fail(RS_EUNSUPPORTED, "chain_blocks exceeds a row's whole blocks");
        }
      }
      const long long nb = tmax / cfg->block_size;
      if (nb > max_nb) max_nb = nb;
      if (tmax > max_tok_all) max_tok_all = tmax;
    }
    return RS_OK;
  };
  // admission order == trace order and many rows: the rows are checked on the
  // device, where they are being uploaded (read back before the first kernel
  // that reads them); otherwise on the host (threads that also gather them)
  const bool dev_check = ident && N >= (1LL << 16);
  int *d_off = nullptr, *d_ol = nullptr, *d_res = nullptr;
  if (dev_check) {
    int* d_chain = nullptr;
    const int init[2] = {0x7FFFFFFF, 0};
    TRY(dalloc(h, &d_off, R + 1, off.data()));
    TRY(dalloc(h, &d_ol, R, ol.data()));
    TRY(dalloc(h, &d_chain, R, chain.data()));
    TRY(dalloc(h, &d_res, 2, init));
    if (R > 0) {
      const int grid = (int)std::min<long long>((R + kWarps - 1) / kWarps, 148 * 8);
      validate_rows_kernel<<<grid, kThreads>>>((int)R, d_off, d_ol, d_chain, d.tok, d.out, cfg->block_size, cfg->cap,
                                               d_res);
      const cudaError_t ke = cudaGetLastError();
      if (ke != cudaSuccess) return fail(RS_ECUDA, std::string("validate_rows_kernel: ") + cudaGetErrorString(ke));
    }
  } else {
    host_scan();
    TRY(check_rows());
  }
  pc.mark("host rows");
  d.R = (int)R;
  d.N = (int)N;
  d.max_size = max_size;
  if (!ident) {
    TRY(dalloc(h, (int**)&d.tok, N, tok));
    TRY(dalloc(h, (int**)&d.out, N, out));
  }
  pc.mark("host rows + arena");
  // unset ledger timestamps: all-ones bytes are a NaN (the host maps any NaN to None)
  TRY(dalloc(h, &d.fps, R, nullptr, 0xFF));
  TRY(dalloc(h, &d.lpe, R, nullptr, 0xFF));
  TRY(dalloc(h, &d.lde, R, nullptr, 0xFF));
  TRY(dalloc(h, &d.gen, N, nullptr, 0));
  TRY(dalloc(h, &d.comp, N, nullptr, 0xFF));
  TRY(dalloc(h, &d.term_spill, (size_t)kMaxJobs * (kSmallMns + 1)));  // scratch: written before read
  {
    std::vector<int> nep(R + 1, 0);  // relQueries with rows among admission ranks [0, a)
    for (long long a = 0; a < R; ++a) nep[a + 1] = nep[a] + (off[a + 1] > off[a]);
    TRY(dalloc(h, (int**)&d.ne_pref, R + 1, nep.data()));
  }
  {
    pc.mark("row uploads");
    // first sight (dpu.cuh first_sight): draw-count prefix on the host, the
    // static PEM of every relQuery by one wide kernel
    std::vector<long long> fsd(R + 1, 0);
    const long long dper = cfg->policy >= RS_POLICY_RELSERVE ? 2 * cfg->sample_size - 1 : 0;
    for (long long a = 0; a < R; ++a) fsd[a + 1] = fsd[a] + ((off[a + 1] - off[a]) > cfg->sample_size ? dper : 0);
    TRY(dalloc(h, (long long**)&d.fs_doff, R + 1, fsd.data()));
    TRY(dalloc(h, (double**)&d.fsprio, R, nullptr, 0));
    if (dev_check) {  // the device row checks (before any kernel reads the rows)
      int res[2];
      const cudaError_t ce = cudaMemcpy(res, d_res, sizeof res, cudaMemcpyDeviceToHost);
      if (ce != cudaSuccess) return fail(RS_ECUDA, std::string("row check readback: ") + cudaGetErrorString(ce));
      if (res[0] != 0x7FFFFFFF) {  // name the offending row (the host checks stop at it)
        host_scan();
        TRY(check_rows());
        return fail(RS_ECUDA, "device row check disagrees with the host");
      }
      max_tok_all = res[1];
      max_nb = max_tok_all / cfg->block_size;
    }
    {
      const long long max_tok = max_tok_all;
      d.seg_ok = cfg->max_num_seqs * max_tok <= cfg->cap && max_tok * kItemBuf < (1LL << 31);
      // engine_kernel<true> (no general DPU path) needs count-only PEM segments,
      // mns and sample size within the warp fast path, and every relQuery's
      // segments within the job buffers
      d.fast = d.seg_ok && cfg->max_num_seqs <= kSmallMns && cfg->sample_size <= 16 &&
               (long long)max_size + cfg->max_num_seqs <= (long long)(kMaxJobs - 1) * cfg->max_num_seqs;
    }
    if (R > 0 && cfg->policy >= RS_POLICY_RELSERVE) {
      if (!d_off) TRY(dalloc(h, &d_off, R + 1, off.data()));
      if (!d_ol) TRY(dalloc(h, &d_ol, R, ol.data()));
      PemModel m{h.pol.alpha_p, h.pol.beta_p, h.pol.alpha_d, h.pol.beta_d, cfg->cap, cfg->max_num_seqs,
                 cfg->max_num_batched_tokens};
      // segment-parallel when segments close by count only and their terms are few
      const long long bound = 2 * cfg->max_num_seqs * max_tok_all / cfg->max_num_batched_tokens + 3;
      const bool seg_fs = d.seg_ok && cfg->max_num_seqs <= kSmallMns && bound <= 64;
      std::vector<int> segp;
      std::vector<int4> segd;  // per segment: first row, rows, output limit
      if (seg_fs) {
        segp.assign(R + 1, 0);
        const int mns = (int)cfg->max_num_seqs;
        for (long long a = 0; a < R; ++a) {
          const int sz = off[a + 1] - off[a];
          segp[a + 1] = segp[a] + (sz + mns - 1) / mns;
          for (int r = 0; r < sz; r += mns) segd.push_back(make_int4(off[a] + r, std::min(mns, sz - r), ol[a], 0));
        }
      }
      int* d_segp = nullptr;
      int4* d_segd = nullptr;
      if (seg_fs) TRY(dalloc(h, &d_segp, R + 1, segp.data()));
      if (seg_fs && !segd.empty()) TRY(dalloc(h, &d_segd, segd.size(), segd.data()));
      const int ns = seg_fs ? segp[R] : 0;
      const int Ri = (int)R;
      const int* tokp = d.tok;
      double* fsp = (double*)d.fsprio;
      auto launch = [=]() -> int {
        if (seg_fs) {
          // terms scratch from the stream-ordered pool, freed after the kernels
          const size_t n_seg = (size_t)std::max(ns, 1);
          const size_t b_terms = n_seg * bound * sizeof(double);
          void* scratch = nullptr;
          if (cudaMallocAsync(&scratch, b_terms + n_seg * 4, 0) != cudaSuccess)
            return fail(RS_ENOMEM, "first-sight scratch");
          double* d_terms = (double*)scratch;
          int* d_nt = (int*)((char*)scratch + b_terms);
          const int grid = (int)std::min<long long>((ns + 255) / 256, 148 * 8);
          if (ns > 0) first_sight_seg_kernel<<<grid, 256>>>(ns, d_segd, tokp, m, (int)bound, d_terms, d_nt);
          first_sight_sum_kernel<<<(unsigned)std::min<long long>((Ri + 255) / 256, 148 * 4), 256>>>(
              Ri, d_segp, (int)bound, d_terms, d_nt, fsp);
          cudaFreeAsync(scratch, 0);
        } else {
          const int grid = (int)std::min<long long>((Ri + kWarps - 1) / kWarps, 148 * 8);
          first_sight_kernel<<<grid, kThreads>>>(Ri, d_off, d_ol, tokp, m, fsp);
        }
        const cudaError_t ke = cudaGetLastError();  // stream-ordered before the static-order sort
        return ke == cudaSuccess ? RS_OK : fail(RS_ECUDA, std::string("first-sight kernels: ") + cudaGetErrorString(ke));
      };
      if (h.deferred) {
        h.pending.push_back(launch);  // after the engine-wide upload (finish_deferred)
      } else {
        TRY(stage_flush(h));  // the kernels read the rows and write fsprio
        TRY(launch());
      }
    }
  }
  pc.mark("first-sight kernel");
  // relQuery table (rq_carve layout), uploaded as one block
  {
    // rank of each rel_id among all rel_ids: the Delta projection's sort key
    std::vector<int> byid(R);
    std::iota(byid.begin(), byid.end(), 0);
    if (!std::is_sorted(relid.begin(), relid.end())) {  // (rel_id, rank) pairs: a stable order
      std::vector<std::pair<long long, int>> kv(R);
      for (long long a = 0; a < R; ++a) kv[a] = {relid[a], (int)a};
      std::sort(kv.begin(), kv.end());
      for (long long i = 0; i < R; ++i) byid[i] = kv[i].second;
    }
    h.rq_host.assign(rq_bytes((int)R) + 16, 0);
    RqView hv = rq_carve(h.rq_host.data(), (int)R);
    for (long long a = 0; a < R; ++a) {
      hv.prio[a] = cfg->policy == RS_POLICY_SP ? sprio[a] : 0.0;  // sp/fcfs priority at admission
      hv.arrival[a] = arrival[a];
      hv.off[a] = off[a];
      hv.ol[a] = ol[a];
      hv.chain[a] = chain[a];
      hv.scr_last[a] = -1;
    }
    hv.off[R] = off[R];
    for (long long i = 0; i < R; ++i) hv.relrank[byid[i]] = (int)i;
    // static waiting order (rq.zl): a never-prefilled relQuery's priority is its
    // first-sight estimate (DPU policies), its static priority (sp) or 0 (fcfs),
    // ordered by (okey(priority), rank) -- the device radix sort at the end of
    // this function (fcfs: every key is 0, the order is the ranks)
    for (long long a = 0; a < R; ++a) hv.zl[a] = (int)a;
    d.nzl = (int)R;
    d.shard_world = shard_world;
    d.shard_rank = shard_rank;
    TRY(dalloc(h, (unsigned char**)&d.rq_global, h.rq_host.size(), h.rq_host.data()));
    h.off.assign(off.begin(), off.end());
  }
  pc.mark("relQuery table");
  // static-order sort scratch (keys, their ping-pong copies, values' ping-pong copy)
  const bool zsort = R > 1 && R <= 0x7FFFFFF0LL && (dpu || cfg->policy == RS_POLICY_SP);
  unsigned long long *zk0 = nullptr, *zk1 = nullptr, *zgh = nullptr;
  int* zv1 = nullptr;
  unsigned* zth = nullptr;
  if (zsort) {
    TRY(dalloc(h, &zk0, R));
    TRY(dalloc(h, &zk1, R));
    TRY(dalloc(h, &zv1, R));
    if (R > kSortOneCta) {  // the grid passes' histograms
      TRY(dalloc(h, &zgh, 8 * 256));
      TRY(dalloc(h, &zth, 256 * ((R + kSortTile - 1) / kSortTile)));
    }
  }
  d.fifo_cap = 1;  // >= capacity + kMaxRun + 2: batched pushes precede evictions
  while (d.fifo_cap < cfg->capacity_blocks + kMaxRun + 2) d.fifo_cap <<= 1;
  TRY(dalloc(h, &d.fifo, d.fifo_cap));  // entries in [head, tail) are written before they are read
  {
    JumpEntry tab[kJumpBits + 32];
    pcg_jump_table(rng, tab);
    pcg_step_table(rng, tab + kJumpBits);
    TRY(dalloc(h, (JumpEntry**)&d.jump, kJumpBits + 32, tab));
  }
  // ring capacities are powers of two so the device indexes them with a mask
  d.log_cap = 0;
  if (log_cap > 0) {
    d.log_cap = 1;
    while (d.log_cap < log_cap) d.log_cap <<= 1;
    TRY(dalloc(h, &d.log, d.log_cap));  // records are written whole before they are read
  } else {  // no log kept: a one-record scratch ring, so the common-configuration kernel (which always
            // writes the record) still applies; status.n_log counts, rs_engine_read_log refuses
    TRY(dalloc(h, &d.log, 1));
    d.log_cap = 1;
    h.no_log = true;
  }
  if (log_cap > 0) {
    if (cfg->record_order) {  // parity mode snapshots (outside the arena: they can be large)
      const size_t cells = (size_t)d.log_cap * std::max<long long>(R, 1);
      TRY(dalloc(h, &d.snap_prio, cells, nullptr, 0xFF));
      TRY(dalloc(h, &d.snap_flag, cells, nullptr, 0));
      TRY(dalloc(h, &d.snap_rng, d.log_cap, nullptr, 0));
    }
  }
  pc.mark("fifo/jump/log");
  Ctl* ctl = (Ctl*)calloc(1, sizeof(Ctl));
  if (!ctl) return fail(RS_ENOMEM, "host alloc");
  ctl->status = RS_RUNNING;
  ctl->rng = rng;
  rc = dalloc(h, &d.ctl, 1, ctl);
  free(ctl);
  if (rc) return rc;
  if (!h.deferred) {
    rc = stage_flush(h);
    h.staging = false;
    std::vector<unsigned char>().swap(h.stage);
    if (rc) return rc;
  }
  pc.mark("uploads");
  // the static waiting order on the device: keys from the first-sight
  // priorities (or sp's static ones in the uploaded table), sorted stably in
  // place into the table's zl section (radix_sort.cuh); stream-ordered after
  // the first-sight kernel and the uploads, no host round trip
  {
    const RqView dv = rq_carve(d.rq_global, (int)R);
    if (zsort) {
      const double* src = dpu ? d.fsprio : dv.prio;
      const int Ri = (int)R;
      auto sort = [=]() -> int {
        static_keys_kernel<<<(unsigned)std::min<long long>((Ri + 255) / 256, 148 * 8), 256>>>(src, Ri, zk0, dv.zl);
        cudaError_t ke = cudaGetLastError();
        if (ke == cudaSuccess) {
          if (Ri <= kSortOneCta) {
            sort_pairs_one_cta<<<1, kSortThreads>>>(zk0, dv.zl, zk1, zv1, Ri);
            ke = cudaGetLastError();
          } else {
            ke = sort_pairs_enqueue(zk0, dv.zl, zk1, zv1, zgh, zth, Ri, 0);
          }
        }
        return ke == cudaSuccess ? RS_OK : fail(RS_ECUDA, std::string("static order sort: ") + cudaGetErrorString(ke));
      };
      if (h.deferred) h.pending.push_back(sort);
      else if ((rc = sort())) return rc;
    }
    if (shard_world > 1) {
      // the full order on the host: a shard keeps the relQueries it owns (shard.cuh),
      // and replicas of this trace on the same device are built from it (clone_replica)
      h.zorder.assign(R, 0);
      if (R) {
        const cudaError_t ce = cudaMemcpy(h.zorder.data(), dv.zl, R * sizeof(int), cudaMemcpyDeviceToHost);
        if (ce != cudaSuccess) return fail(RS_ECUDA, std::string("static order readback: ") + cudaGetErrorString(ce));
      }
    }
    RqView hv = rq_carve(h.rq_host.data(), (int)R);
    int nz = 0;
    for (long long i = 0; i < (long long)h.zorder.size(); ++i)
      if (h.zorder[i] % shard_world == shard_rank) hv.zl[nz++] = h.zorder[i];
    if (shard_world > 1) {
      d.nzl = nz;
      const cudaError_t ce = cudaMemcpy(dv.zl, hv.zl, (size_t)nz * sizeof(int), cudaMemcpyHostToDevice);
      if (ce != cudaSuccess) return fail(RS_ECUDA, std::string("shard static order: ") + cudaGetErrorString(ce));
    }
  }
  pc.mark("static order");
#undef TRY
  return RS_OK;
}

// Another shard's replica of a built trace (sharded pool, all shards in one
// engine): the read-only columns (tok, out, first-sight priorities and draw
// offsets, the RNG jump tables) are shared with `src`; the mutable state gets
// its own arena, initialised as build_trace does, and the relQuery table its
// shard's static waiting order.
static int clone_replica(const HostTrace& src, const rs_config* cfg, const rs_pcg64_state& rng, HostTrace& h,
                         int shard_world, int shard_rank) {
  h.pol = src.pol;
  h.off = src.off;
  h.rank_of = src.rank_of;
  h.order = src.order;
  h.row_src = src.row_src;
  h.zorder = src.zorder;
  h.rq_host = src.rq_host;
  h.dev = src.dev;
  TraceDev& d = h.dev;
  const long long R = d.R, N = d.N;
  int rc;
#define TRY(x) \
  if ((rc = (x))) return rc
  const size_t need = 8 * (size_t)N + 24 * (size_t)R + 8 * (size_t)kMaxJobs * (kSmallMns + 1) + rq_bytes((int)R) +
                      16 + (size_t)d.fifo_cap * sizeof(FifoEnt) + (size_t)d.log_cap * sizeof(rs_iter_record) +
                      sizeof(Ctl) + 16 * 256;
  TRY(arena_reserve(h, need));
  // unset ledger timestamps: all-ones bytes are a NaN (the host maps any NaN to None)
  TRY(dalloc(h, &d.fps, R, nullptr, 0xFF));
  TRY(dalloc(h, &d.lpe, R, nullptr, 0xFF));
  TRY(dalloc(h, &d.lde, R, nullptr, 0xFF));
  TRY(dalloc(h, &d.gen, N, nullptr, 0));
  TRY(dalloc(h, &d.comp, N, nullptr, 0xFF));
  TRY(dalloc(h, &d.term_spill, (size_t)kMaxJobs * (kSmallMns + 1)));  // scratch: written before read
  {
    // the host columns are shard 0's (shared, not copied); only this shard's static order differs
    const int* zo = h.zorder.cdata();
    std::vector<int> zl;
    zl.reserve((size_t)(R / shard_world + 1));
    for (long long i = 0; i < R; ++i)
      if (zo[i] % shard_world == shard_rank) zl.push_back(zo[i]);
    d.nzl = (int)zl.size();
    d.shard_world = shard_world;
    d.shard_rank = shard_rank;
    // the table is shard 0's (device to device) but for this shard's static order
    TRY(dalloc(h, (unsigned char**)&d.rq_global, h.rq_host.size()));
    const unsigned char* base = h.rq_host.cdata();
    const size_t zl_at = (size_t)((const unsigned char*)rq_carve(const_cast<unsigned char*>(base), (int)R).zl - base);
    if (cudaMemcpyAsync(d.rq_global, src.dev.rq_global, h.rq_host.size(), cudaMemcpyDeviceToDevice, 0) != cudaSuccess ||
        (!zl.empty() && cudaMemcpy((unsigned char*)d.rq_global + zl_at, zl.data(), zl.size() * sizeof(int),
                                   cudaMemcpyHostToDevice) != cudaSuccess))
      return fail(RS_ECUDA, "replica relQuery table copy failed");
  }
  TRY(dalloc(h, &d.fifo, d.fifo_cap));  // entries in [head, tail) are written before they are read
  if (d.log_cap > 0) TRY(dalloc(h, &d.log, d.log_cap));
  Ctl* ctl = (Ctl*)calloc(1, sizeof(Ctl));
  if (!ctl) return fail(RS_ENOMEM, "host alloc");
  ctl->status = RS_RUNNING;
  ctl->rng = rng;
  rc = dalloc(h, &d.ctl, 1, ctl);
  free(ctl);
#undef TRY
  return rc;
}

static int upload_traces(rs_engine* e) {
  const int n = (int)e->traces.size();
  std::vector<TraceDev> devs(n);
  for (int t = 0; t < n; ++t) devs[t] = e->traces[t].dev;
  if (!e->d_traces && cudaMallocAsync(&e->d_traces, sizeof(TraceDev) * n, 0) != cudaSuccess)
    return fail(RS_ECUDA, "trace table allocation failed");
  if (cudaMemcpy(e->d_traces, devs.data(), sizeof(TraceDev) * n, cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(RS_ECUDA, "trace table upload failed");
  return RS_OK;
}

// The deferred small traces (build_trace): their staged arena images go up in
// one page-locked batch of asynchronous copies, then each trace's creation
// kernels (first sight, static-order sort) are launched, all stream-ordered on
// the legacy stream -- no host round trip per trace.
static int finish_deferred(rs_engine* e, bool with_table) {
  size_t total = 0;
  for (auto& h : e->traces)
    if (h.deferred) total += h.arena_used - h.staged_lo;
  const size_t table = with_table ? ((sizeof(TraceDev) * e->traces.size() + 255) & ~(size_t)255) : 0;
  if (with_table) {
    total += table;
    if (!e->d_traces && cudaMallocAsync(&e->d_traces, sizeof(TraceDev) * e->traces.size(), 0) != cudaSuccess)
      return fail(RS_ECUDA, "trace table allocation failed");
  }
  if (total) {
    std::lock_guard<std::mutex> lk(g_pinned.mu);
    if (g_pinned.done) cudaEventSynchronize(g_pinned.done);  // the previous creation's copies are done
    if (g_pinned.cap < total) {
      if (g_pinned.p) cudaFreeHost(g_pinned.p);
      g_pinned.p = nullptr;
      g_pinned.cap = 0;
      const size_t want = total + total / 4 + (1 << 20);
      if (cudaMallocHost((void**)&g_pinned.p, want) == cudaSuccess) g_pinned.cap = want;
    }
    size_t o = 0;
    if (with_table) {  // the trace table (every pointer is final once the traces are built)
      for (size_t t = 0; t < e->traces.size(); ++t) {
        if (g_pinned.p) memcpy(g_pinned.p + t * sizeof(TraceDev), &e->traces[t].dev, sizeof(TraceDev));
      }
      const cudaError_t ce =
          g_pinned.p ? cudaMemcpyAsync(e->d_traces, g_pinned.p, sizeof(TraceDev) * e->traces.size(),
                                       cudaMemcpyHostToDevice, 0)
                     : cudaSuccess;
      if (ce != cudaSuccess) return fail(RS_ECUDA, std::string("trace table upload: ") + cudaGetErrorString(ce));
      o += table;
    }
    for (auto& h : e->traces) {
      if (!h.deferred) continue;
      const size_t n = h.arena_used - h.staged_lo;
      if (!n) continue;
      cudaError_t ce;
      if (g_pinned.p) {
        memcpy(g_pinned.p + o, h.stage.data() + h.staged_lo, n);
        ce = cudaMemcpyAsync(h.arena + h.staged_lo, g_pinned.p + o, n, cudaMemcpyHostToDevice, 0);
        o += n;
      } else {  // no page-locked memory: a staged copy per trace
        ce = cudaMemcpy(h.arena + h.staged_lo, h.stage.data() + h.staged_lo, n, cudaMemcpyHostToDevice);
      }
      if (ce != cudaSuccess) return fail(RS_ECUDA, std::string("deferred upload: ") + cudaGetErrorString(ce));
      h.staged_lo = h.arena_used;
    }
    if (g_pinned.p) {
      if (!g_pinned.done) cudaEventCreateWithFlags(&g_pinned.done, cudaEventDisableTiming);
      cudaEventRecord(g_pinned.done, 0);
    }
  }
  if (with_table && !g_pinned.p) {  // no page-locked memory: the synchronous path
    const int rc = upload_traces(e);
    if (rc) return rc;
  }
  for (auto& h : e->traces) {
    if (!h.deferred) continue;
    h.staging = false;
    std::vector<unsigned char>().swap(h.stage);
    for (auto& f : h.pending) {
      const int rc = f();
      if (rc) return rc;
    }
    h.pending.clear();
    h.deferred = false;
  }
  // creation returns without waiting: the first launch (or status read) waits for this
  if (!e->ready && cudaEventCreateWithFlags(&e->ready, cudaEventDisableTiming) != cudaSuccess)
    return fail(RS_ECUDA, "creation event");
  if (cudaEventRecord(e->ready, 0) != cudaSuccess) return fail(RS_ECUDA, "creation event record");
  return RS_OK;
}


// shard_world == 1: independent traces.  shard_world > 1: every trace is a
// replica of one trace; replica t is shard t when shard_rank == -1 (all
// shards in this engine), else the single replica is shard `shard_rank`.
static int create_impl(const rs_trace_view* traces, int32_t n_traces, const rs_config* cfg,
                       const rs_cost_model* world, const rs_cost_model* policy_model, const rs_pcg64_state* rng,
                       int32_t device, int64_t log_capacity, int shard_world, int shard_rank, rs_engine** out) {
  *out = nullptr;
  if (n_traces <= 0) return fail(RS_EINVAL, "n_traces must be positive");
  int rc = validate_config(cfg);
  if (rc) return rc;
  PhaseClock pc;
  RS_CUDA(cudaSetDevice(device));
  keep_pool(device);
  pc.mark("cudaSetDevice");
  rs_engine* e = new rs_engine();
  e->device = device;
  e->shard_world = shard_world;
  e->shard_rank = shard_rank;
  e->traces.resize(n_traces);
  auto bail = [&](int code) {
    std::string keep = g_err;
    rs_engine_destroy(e);
    g_err = keep;
    return code;
  };
  if (shard_world == 1 && n_traces > 1) {  // independent traces: one arena, sliced (one allocation)
    std::vector<size_t> needs(n_traces);
    size_t total = 0;
    for (int t = 0; t < n_traces; ++t) total += needs[t] = arena_need(traces[t], cfg, log_capacity);
    void* q = nullptr;
    if (cudaMallocAsync(&q, total, 0) != cudaSuccess) return bail(fail(RS_ENOMEM, "engine arena"));
    size_t o = 0;
    for (int t = 0; t < n_traces; ++t) {
      HostTrace& h = e->traces[t];
      h.arena_alloc = t == 0 ? q : nullptr;  // trace 0 owns (frees) the allocation
      h.arena = (char*)q + o;
      h.arena_cap = needs[t];
      o += needs[t];
    }
  }
  for (int t = 0; t < n_traces; ++t) {
    const int srank = shard_world == 1 ? 0 : (shard_rank < 0 ? t : shard_rank);
    if (shard_world > 1 && shard_rank < 0 && t > 0)  // another shard of the same pool on this device
      rc = clone_replica(e->traces[0], cfg, rng[t], e->traces[t], shard_world, srank);
    else
      rc = build_trace(traces[t], cfg, *policy_model, rng[t], log_capacity, e->traces[t], shard_world, srank);
    if (rc) return bail(rc);
    if (shard_world > 1) pc.mark(t == 0 ? "shard 0 built" : "replica cloned");
  }
  // shared memory: the control block etc., plus the relQuery table of every
  // trace whose table fits next to it (the others read theirs from HBM)
  const size_t base = (sizeof(Shared) + 15) & ~(size_t)15;
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  size_t need = base;
  for (auto& h : e->traces) {
    const size_t rb = rq_bytes(h.dev.R);
    h.dev.rq_in_smem = base + rb <= (size_t)max_optin;
    if (h.dev.rq_in_smem) need = std::max(need, base + rb);
  }
  bool all_deferred = shard_world == 1;
  for (auto& h : e->traces) all_deferred = all_deferred && h.deferred;
  if ((rc = finish_deferred(e, all_deferred))) return bail(rc);
  pc.mark("deferred uploads");
  if (shard_world > 1) {  // mailboxes (shard.cuh); zeroed: sequence numbers start at 1
    const size_t mb = mailbox_bytes(shard_world);
    const int n_mb = shard_rank < 0 ? shard_world : 1;
    // one process: from the stream-ordered pool (a plain cudaMalloc here measured 3-30 ms next to
    // torch's cached allocations); one shard per process: cudaMalloc, the mailbox is IPC-exported
    e->mbox_pooled = shard_rank < 0;
    const cudaError_t am = e->mbox_pooled ? cudaMallocAsync(&e->mbox, mb * n_mb, 0) : cudaMalloc(&e->mbox, mb * n_mb);
    if (am != cudaSuccess || cudaMemsetAsync(e->mbox, 0, mb * n_mb, 0) != cudaSuccess ||
        cudaMallocAsync(&e->d_peers, sizeof(ShardRec*) * shard_world, 0) != cudaSuccess)
      return bail(fail(RS_ENOMEM, "mailbox allocation failed"));
    std::vector<ShardRec*> peers(shard_world, nullptr);
    for (int d = 0; d < shard_world; ++d)
      peers[d] = shard_rank < 0 ? (ShardRec*)((char*)e->mbox + mb * d) : (d == shard_rank ? e->mbox : nullptr);
    if (cudaMemcpy(e->d_peers, peers.data(), sizeof(ShardRec*) * shard_world, cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(RS_ECUDA, "mailbox table upload failed"));
    for (int t = 0; t < n_traces; ++t) {
      e->traces[t].dev.self_mbox = shard_rank < 0 ? peers[t] : e->mbox;
      e->traces[t].dev.peers = e->d_peers;
    }
    e->connected = shard_rank < 0;
  }
  pc.mark("traces built");
  if (!all_deferred && (rc = upload_traces(e))) return bail(rc);
  pc.mark("trace table");
  Params& p = e->params;
  p.traces = e->d_traces;
  p.cfg = *cfg;
  p.world = *world;
  p.pol = *policy_model;
  p.use_dpu = cfg->policy >= RS_POLICY_RELSERVE;
  p.force = cfg->policy == RS_POLICY_RELSERVE_PP ? 1 : cfg->policy == RS_POLICY_RELSERVE_DP ? 2 : 0;
  p.prefill_first = cfg->policy == RS_POLICY_FCFS || cfg->policy == RS_POLICY_SP;
  p.zorder = !p.use_dpu || std::isinf(cfg->tau);
  p.mns_magic = (unsigned long long)(0xFFFFFFFFull / (unsigned long long)cfg->max_num_seqs) + 1;  // see dpu_small
  p.dper_magic = (unsigned)(65536 / std::max<long long>(1, 2 * cfg->sample_size - 1)) + 1;
  e->smem = need;
  e->fast = true;
  for (auto& h : e->traces) e->fast = e->fast && h.dev.fast;
  // the common configuration's specialised kernel (see iterate)
  e->common = e->fast && p.use_dpu && std::isinf(cfg->tau) && !(cfg->noise_sigma > 0) && cfg->log_decisions &&
              cfg->block_size == 16 && cfg->sample_size == 8;
  for (auto& h : e->traces) e->common = e->common && h.dev.log_cap > 0;
  e->part = false;  // a relQuery table in HBM (large traces: long re-estimate lists are common)
  for (auto& h : e->traces) e->part = e->part || !h.dev.rq_in_smem;
  // the kernels' dynamic shared-memory limit only grows (engines with different needs may coexist);
  // the L1/shared carve-out is left to the driver, which sizes it by each launch's request
  static std::mutex attr_mu;
  static size_t smem_limit = 0;
  cudaError_t ce = cudaSuccess;
  {
    std::lock_guard<std::mutex> lk(attr_mu);
    const size_t lim = std::max(smem_limit, e->smem);
    ce = cudaFuncSetAttribute(engine_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim);
    if (ce == cudaSuccess)
      ce = cudaFuncSetAttribute(engine_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim);
    if (ce == cudaSuccess)
      ce = cudaFuncSetAttribute(engine_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim);
    if (ce == cudaSuccess)
      ce = cudaFuncSetAttribute(engine_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim);
#ifdef RS_CARVEOUT  // experiment: ask for the smallest carve-out that holds this engine's shared memory
    const int pct = (int)std::min<size_t>(100, (e->smem + 1024) * 100 / (228 * 1024) + 1);
    if (ce == cudaSuccess)
      ce = cudaFuncSetAttribute(engine_kernel<true, true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
#endif
    if (ce == cudaSuccess) smem_limit = lim;
  }
  if (ce != cudaSuccess) return bail(fail(RS_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(ce)));
  pc.mark("kernel attributes");
  *out = e;
  return RS_OK;
}

int rs_engine_create(const rs_trace_view* traces, int32_t n_traces, const rs_config* cfg,
                     const rs_cost_model* world, const rs_cost_model* policy_model,
                     const rs_pcg64_state* rng, int32_t device, int64_t log_capacity, rs_engine** out) {
  return create_impl(traces, n_traces, cfg, world, policy_model, rng, device, log_capacity, 1, 0, out);
}

int rs_engine_create_sharded(const rs_trace_view* trace, const rs_config* cfg, const rs_cost_model* world,
                             const rs_cost_model* policy_model, const rs_pcg64_state* rng, int32_t device,
                             int64_t log_capacity, int32_t shards, int32_t rank, rs_engine** out) {
  *out = nullptr;
  if (shards < 1 || shards > 32) return fail(RS_EINVAL, "shards must be in [1, 32]");
  if (rank < -1 || rank >= shards) return fail(RS_EINVAL, "rank must be -1 or in [0, shards)");
  int n_sm = 0;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device);
  if (rank < 0 && shards > n_sm) return fail(RS_EINVAL, "all-shards-here mode needs one SM per shard");
  const int n = rank < 0 ? shards : 1;
  std::vector<rs_trace_view> views(n, *trace);
  std::vector<rs_pcg64_state> rngs(n, *rng);
  return create_impl(views.data(), n, cfg, world, policy_model, rngs.data(), device, log_capacity, shards,
                     shards == 1 ? 0 : rank, out);
}

int rs_engine_mailbox(rs_engine* e, void** dptr, int64_t* bytes) {
  if (!e || e->shard_world < 2 || e->shard_rank < 0) return fail(RS_EINVAL, "not a one-shard sharded engine");
  *dptr = e->mbox;
  *bytes = (int64_t)mailbox_bytes(e->shard_world);
  return RS_OK;
}

int rs_engine_connect(rs_engine* e, void* const* peer_mailboxes) {
  if (!e || e->shard_world < 2 || e->shard_rank < 0) return fail(RS_EINVAL, "not a one-shard sharded engine");
  RS_CUDA(cudaSetDevice(e->device));
  std::vector<ShardRec*> peers(e->shard_world);
  for (int d = 0; d < e->shard_world; ++d) {
    peers[d] = d == e->shard_rank ? e->mbox : (ShardRec*)peer_mailboxes[d];
    if (!peers[d]) return fail(RS_EINVAL, "null peer mailbox");
  }
  RS_CUDA(cudaMemcpy(e->d_peers, peers.data(), sizeof(ShardRec*) * e->shard_world, cudaMemcpyHostToDevice));
  e->connected = true;
  return RS_OK;
}

int rs_ipc_get_handle(void* dptr, uint8_t* handle) {
  cudaIpcMemHandle_t h;
  RS_CUDA(cudaIpcGetMemHandle(&h, dptr));
  memcpy(handle, &h, sizeof h);
  return RS_OK;
}

int rs_ipc_open_handle(const uint8_t* handle, int32_t device, void** dptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  RS_CUDA(cudaSetDevice(device));
  RS_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return RS_OK;
}

int rs_ipc_close(void* dptr) {
  RS_CUDA(cudaIpcCloseMemHandle(dptr));
  return RS_OK;
}

int rs_engine_set_noise(rs_engine* e, int32_t t, const double* z, int64_t n) {
  if (!e || t < -1 || t >= (int)e->traces.size()) return fail(RS_EINVAL, "bad trace index");
  if (n < 0 || (n > 0 && !z)) return fail(RS_EINVAL, "bad noise buffer");
  RS_CUDA(cudaSetDevice(e->device));
  for (int i = 0; i < (int)e->traces.size(); ++i) {
    if (t >= 0 && i != t) continue;
    HostTrace& h = e->traces[i];
    double* d = nullptr;
    RS_CUDA(cudaMalloc(&d, std::max<int64_t>(n, 1) * sizeof(double)));
    if (n) RS_CUDA(cudaMemcpy(d, z, n * sizeof(double), cudaMemcpyHostToDevice));
    if (h.noise_buf) cudaFree(h.noise_buf);
    h.noise_buf = d;
    h.dev.noise = d;
    h.dev.noise_n = n;
  }
  return upload_traces(e);
}

int rs_engine_step(rs_engine* e, int64_t max_iters, void* stream) {
  if (!e) return fail(RS_EINVAL, "null engine");
  if (e->params.cfg.noise_sigma > 0)
    for (auto& h : e->traces)
      if (!h.noise_buf) return fail(RS_EINVAL, "noise_sigma > 0 needs rs_engine_set_noise before stepping");
  if (e->shard_world > 1 && !e->connected) return fail(RS_EINVAL, "sharded engine not connected to its peers");
  RS_CUDA(cudaSetDevice(e->device));
  // a launch writes at most one ring of records (the host reads them between launches)
  const bool logs = e->params.cfg.log_decisions && !e->traces[0].no_log;
  const long long cap = logs ? e->traces[0].dev.log_cap : max_iters;
  if (logs && cap > 0 && max_iters > cap) max_iters = cap;
  if (e->ready) RS_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, e->ready, 0));  // creation's uploads / kernels
  Params p = e->params;
  p.max_iters = max_iters;
  if (e->common && e->part)
    engine_kernel<true, true, true><<<(unsigned)e->traces.size(), kThreads, e->smem, (cudaStream_t)stream>>>(p);
  else if (e->common)
    engine_kernel<true, true><<<(unsigned)e->traces.size(), kThreads, e->smem, (cudaStream_t)stream>>>(p);
  else if (e->fast)
    engine_kernel<true, false><<<(unsigned)e->traces.size(), kThreads, e->smem, (cudaStream_t)stream>>>(p);
  else
    engine_kernel<false, false><<<(unsigned)e->traces.size(), kThreads, e->smem, (cudaStream_t)stream>>>(p);
  RS_CUDA(cudaGetLastError());
  if (!e->done) RS_CUDA(cudaEventCreateWithFlags(&e->done, cudaEventDisableTiming));
  RS_CUDA(cudaEventRecord(e->done, (cudaStream_t)stream));
  return RS_OK;
}

int rs_engine_status(rs_engine* e, void* stream, rs_trace_status* st) {
  if (!e) return fail(RS_EINVAL, "null engine");
  RS_CUDA(cudaSetDevice(e->device));
  // every trace's control-block header into page-locked memory, ordered after the
  // stream's launches, then one synchronisation
  const size_t head = (offsetof(Ctl, run_row) + 15) & ~(size_t)15;
  const size_t total = head * e->traces.size();
  static std::mutex mu;
  static unsigned char* buf = nullptr;
  static size_t cap = 0;
  std::lock_guard<std::mutex> lk(mu);
  if (cap < total) {
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    cap = 0;
    RS_CUDA(cudaMallocHost((void**)&buf, std::max<size_t>(total, 64 << 10)));
    cap = std::max<size_t>(total, 64 << 10);
  }
  const cudaStream_t strm = (cudaStream_t)stream;
  if (e->ready) RS_CUDA(cudaStreamWaitEvent(strm, e->ready, 0));
  for (size_t t = 0; t < e->traces.size(); ++t)
    RS_CUDA(cudaMemcpyAsync(buf + t * head, e->traces[t].dev.ctl, offsetof(Ctl, run_row), cudaMemcpyDeviceToHost,
                            strm));
  RS_CUDA(cudaStreamSynchronize(strm));
  for (size_t t = 0; t < e->traces.size(); ++t) {
    const Ctl* c = reinterpret_cast<const Ctl*>(buf + t * head);
    rs_trace_status& s = st[t];
    s.iterations = c->iteration;
    s.clock = c->clock;
    s.cache_hit_tokens = c->hit;
    s.cache_miss_tokens = c->miss;
    s.kv_reserved = c->kv;
    s.n_log = c->n_log;
    s.live_relqueries = c->live;
    s.admitted = c->n_admitted;
    s.status = c->status;
    s.error_detail = c->error_detail;
    s.rng = c->rng;
    for (int k = 0; k < 23; ++k) s.phase_cycles[k] = c->phase[k];
    s.alg_bytes = c->alg_bytes;
    s.batches = c->n_batch;
  }
  return RS_OK;
}

int rs_engine_read_log(rs_engine* e, int32_t t, int64_t first, int64_t count, rs_iter_record* out) {
  if (!e || t < 0 || t >= (int)e->traces.size()) return fail(RS_EINVAL, "bad trace index");
  const TraceDev& d = e->traces[t].dev;
  if (count <= 0) return RS_OK;
  if (e->traces[t].no_log) return fail(RS_EINVAL, "engine created without a decision log (log_capacity 0)");
  if (d.log_cap <= 0 || count > d.log_cap) return fail(RS_EINVAL, "log range exceeds the ring buffer");
  RS_CUDA(cudaSetDevice(e->device));
  long long done = 0;
  while (done < count) {
    const long long pos = (first + done) % d.log_cap;
    const long long n = std::min(count - done, d.log_cap - pos);
    RS_CUDA(cudaMemcpy(out + done, d.log + pos, n * sizeof(rs_iter_record), cudaMemcpyDeviceToHost));
    done += n;
  }
  // records carry rank indices; map to trace-order indices
  const HostTrace& h = e->traces[t];
  for (long long i = 0; i < count; ++i) {
    if (out[i].head >= 0) out[i].head = h.order[out[i].head];
    if (out[i].batch_rq >= 0) out[i].batch_rq = h.order[out[i].batch_rq];
  }
  return RS_OK;
}

// Parity-mode readers.  Row i of every output is the snapshot of iteration
// first + i (the ring must still hold it: count <= log capacity, read before
// the next launch).
static int parity_rows(rs_engine* e, int32_t t, int64_t first, int64_t count, const HostTrace** hp) {
  if (!e || t < 0 || t >= (int)e->traces.size()) return fail(RS_EINVAL, "bad trace index");
  const HostTrace& h = e->traces[t];
  if (!h.dev.snap_prio) return fail(RS_EINVAL, "engine created without record_order (parity mode)");
  if (count < 0 || count > h.dev.log_cap) return fail(RS_EINVAL, "range exceeds the parity ring");
  *hp = &h;
  return RS_OK;
}

int rs_engine_read_dpu(rs_engine* e, int32_t t, int64_t first, int64_t count, double* values, uint8_t* flags,
                       rs_pcg64_state* rng) {
  const HostTrace* hp = nullptr;
  int rc = parity_rows(e, t, first, count, &hp);
  if (rc) return rc;
  const HostTrace& h = *hp;
  const TraceDev& d = h.dev;
  const long long R = d.R;
  RS_CUDA(cudaSetDevice(e->device));
  std::vector<double> vb(R);
  std::vector<unsigned char> fb(R);
  for (long long i = 0; i < count; ++i) {
    const long long row = (first + i) & (d.log_cap - 1);
    if (values || flags) {
      RS_CUDA(cudaMemcpy(vb.data(), d.snap_prio + row * R, R * sizeof(double), cudaMemcpyDeviceToHost));
      RS_CUDA(cudaMemcpy(fb.data(), d.snap_flag + row * R, R, cudaMemcpyDeviceToHost));
      for (long long a = 0; a < R; ++a) {  // ranks -> trace order
        if (values) values[i * R + h.order[a]] = vb[a];
        if (flags) flags[i * R + h.order[a]] = fb[a];
      }
    }
    if (rng) RS_CUDA(cudaMemcpy(rng + i, d.snap_rng + row, sizeof(rs_pcg64_state), cudaMemcpyDeviceToHost));
  }
  return RS_OK;
}

}  // extern "C"

namespace {

// per parity row: the number of waiting relQueries (pass 1) / their (key, rank) at off[i] (pass 2)
__global__ void __launch_bounds__(kThreads) parity_gather_kernel(const double* snap_prio, const unsigned char* snap_flag,
                                                                 long long R, long long first, long long mask,
                                                                 const long long* off, int* cnt,
                                                                 unsigned long long* key, int* idx, int* rank,
                                                                 unsigned long long* rowk) {
  __shared__ Scan32Smem s32;
  const long long row = (first + blockIdx.x) & mask;
  const unsigned char* f = snap_flag + row * R;
  const double* v = snap_prio + row * R;
  long long base = off ? off[blockIdx.x] : 0;
  int n = 0;
  for (long long a0 = 0; a0 < R; a0 += kThreads) {
    const long long a = a0 + threadIdx.x;
    const bool w = a < R && (f[a] & kSnapWaiting);
    int x[1] = {w ? 1 : 0}, tot[1];
    block_scan32<1>(x, s32, tot);
    if (off && w) {
      const long long e = base + n + x[0] - 1;
      key[e] = okey(v[a]);
      idx[e] = (int)e;
      rank[e] = (int)a;
      rowk[e] = (unsigned long long)blockIdx.x;
    }
    n += tot[0];
  }
  if (!off && threadIdx.x == 0) cnt[blockIdx.x] = n;
}

__global__ void parity_rowkeys_kernel(const unsigned long long* rowk, const int* idx, unsigned long long* key2,
                                      long long n) {
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
    key2[j] = rowk[idx[j]];
}

__global__ void parity_ranks_kernel(const int* rank, const int* idx, int* out, long long n) {
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
    out[j] = rank[idx[j]];
}

}  // namespace

extern "C" {

int rs_engine_read_order(rs_engine* e, int32_t t, int64_t first, int64_t count, int32_t* out) {
  const HostTrace* hp = nullptr;
  int rc = parity_rows(e, t, first, count, &hp);
  if (rc) return rc;
  if (count == 0) return RS_OK;
  const HostTrace& h = *hp;
  const TraceDev& d = h.dev;
  const long long R = d.R;
  RS_CUDA(cudaSetDevice(e->device));
  for (long long i = 0; i < count * R; ++i) out[i] = -1;
  if (R == 0) return RS_OK;
  DevBuf b;
  int* cnt = nullptr;
  long long* off = nullptr;
  RS_CUDA(b.get(&cnt, count));
  RS_CUDA(b.get(&off, count + 1));
  parity_gather_kernel<<<(unsigned)count, kThreads>>>(d.snap_prio, d.snap_flag, R, first, d.log_cap - 1, nullptr, cnt,
                                                      nullptr, nullptr, nullptr, nullptr);
  RS_CUDA(cudaGetLastError());
  std::vector<int> hc(count);
  RS_CUDA(cudaMemcpy(hc.data(), cnt, count * 4, cudaMemcpyDeviceToHost));
  std::vector<long long> ho(count + 1, 0);
  for (long long i = 0; i < count; ++i) ho[i + 1] = ho[i] + hc[i];
  const long long n = ho[count];
  if (n == 0) return RS_OK;
  if (n > 0x7FFFFFF0LL) return fail(RS_EUNSUPPORTED, "parity order read too large; read fewer rows");
  RS_CUDA(cudaMemcpy(off, ho.data(), (count + 1) * 8, cudaMemcpyHostToDevice));
  unsigned long long *key = nullptr, *rowk = nullptr;
  int *idx = nullptr, *rank = nullptr, *res = nullptr;
  RS_CUDA(b.get(&key, n));
  RS_CUDA(b.get(&rowk, n));
  RS_CUDA(b.get(&idx, n));
  RS_CUDA(b.get(&rank, n));
  RS_CUDA(b.get(&res, n));
  parity_gather_kernel<<<(unsigned)count, kThreads>>>(d.snap_prio, d.snap_flag, R, first, d.log_cap - 1, off, cnt, key,
                                                      idx, rank, rowk);
  RS_CUDA(cudaGetLastError());
  // (priority key, rank) order within each row: stable by key from rank order, then stable by row
  if ((rc = sort_pairs_dev(key, idx, n, 0))) return rc;
  parity_rowkeys_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 8), 256>>>(rowk, idx, key, n);
  if ((rc = sort_pairs_dev(key, idx, n, 0))) return rc;
  parity_ranks_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 8), 256>>>(rank, idx, res, n);
  RS_CUDA(cudaGetLastError());
  std::vector<int> hr(n);
  RS_CUDA(cudaMemcpy(hr.data(), res, n * 4, cudaMemcpyDeviceToHost));
  for (long long i = 0; i < count; ++i)
    for (long long j = ho[i]; j < ho[i + 1]; ++j) out[i * R + (j - ho[i])] = h.order[hr[j]];
  return RS_OK;
}

int rs_engine_read_results(rs_engine* e, void* stream, double* fps, double* lpe, double* lde, int32_t* completion_iter) {
  if (!e) return fail(RS_EINVAL, "null engine");
  RS_CUDA(cudaSetDevice(e->device));
  // every trace's device columns into one page-locked buffer, one synchronisation
  size_t total = 0;
  for (auto& h : e->traces) total += 24 * (size_t)h.dev.R + 4 * (size_t)h.dev.N;
  static std::mutex mu;
  static unsigned char* buf = nullptr;
  static size_t cap = 0;
  std::lock_guard<std::mutex> lk(mu);
  if (cap < total) {
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    cap = 0;
    RS_CUDA(cudaMallocHost((void**)&buf, total + total / 4 + 4096));
    cap = total + total / 4 + 4096;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (e->ready) RS_CUDA(cudaStreamWaitEvent(st, e->ready, 0));
  size_t o = 0;
  for (auto& h : e->traces) {
    const TraceDev& d = h.dev;
    if (d.R) {
      RS_CUDA(cudaMemcpyAsync(buf + o, d.fps, 8 * (size_t)d.R, cudaMemcpyDeviceToHost, st));
      RS_CUDA(cudaMemcpyAsync(buf + o + 8 * (size_t)d.R, d.lpe, 8 * (size_t)d.R, cudaMemcpyDeviceToHost, st));
      RS_CUDA(cudaMemcpyAsync(buf + o + 16 * (size_t)d.R, d.lde, 8 * (size_t)d.R, cudaMemcpyDeviceToHost, st));
    }
    if (d.N) RS_CUDA(cudaMemcpyAsync(buf + o + 24 * (size_t)d.R, d.comp, 4 * (size_t)d.N, cudaMemcpyDeviceToHost, st));
    o += 24 * (size_t)d.R + 4 * (size_t)d.N;
  }
  RS_CUDA(cudaStreamSynchronize(st));
  // ranks -> trace order, traces concatenated
  o = 0;
  size_t ro = 0, no = 0;
  for (auto& h : e->traces) {
    const int R = h.dev.R, N = h.dev.N;
    const double* b = (const double*)(buf + o);
    for (int a = 0; a < R; ++a) {
      const size_t i = ro + h.order[a];
      if (fps) fps[i] = b[a];
      if (lpe) lpe[i] = b[R + a];
      if (lde) lde[i] = b[2 * R + a];
    }
    const int* cp = (const int*)(buf + o + 24 * (size_t)R);
    if (completion_iter) {
      if (h.row_src.empty()) memcpy(completion_iter + no, cp, 4 * (size_t)N);
      else
        for (int k = 0; k < N; ++k) completion_iter[no + h.row_src[k]] = cp[k];
    }
    o += 24 * (size_t)R + 4 * (size_t)N;
    ro += R;
    no += N;
  }
  return RS_OK;
}

int rs_engine_read_ledgers(rs_engine* e, int32_t t, double* arrival, double* fps, double* lpe, double* lde) {
  if (!e || t < 0 || t >= (int)e->traces.size()) return fail(RS_EINVAL, "bad trace index");
  const HostTrace& h = e->traces[t];
  const int R = h.dev.R;
  RS_CUDA(cudaSetDevice(e->device));
  std::vector<double> b(R), c(R), d(R);
  if (R) {
    RS_CUDA(cudaMemcpy(b.data(), h.dev.fps, R * 8, cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(c.data(), h.dev.lpe, R * 8, cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(d.data(), h.dev.lde, R * 8, cudaMemcpyDeviceToHost));
  }
  const RqView hv = rq_carve(const_cast<unsigned char*>(h.rq_host.cdata()), R);
  for (int r = 0; r < R; ++r) {
    const int i = h.order[r];
    if (arrival) arrival[i] = hv.arrival[r];
    if (fps) fps[i] = b[r];
    if (lpe) lpe[i] = c[r];
    if (lde) lde[i] = d[r];
  }
  return RS_OK;
}

int rs_engine_read_requests(rs_engine* e, int32_t t, int32_t* generated, uint8_t* prefilled,
                            int64_t* completion_iter, double* priority) {
  if (!e || t < 0 || t >= (int)e->traces.size()) return fail(RS_EINVAL, "bad trace index");
  const HostTrace& h = e->traces[t];
  const int R = h.dev.R, N = h.dev.N;
  RS_CUDA(cudaSetDevice(e->device));
  if (h.row_src.empty() && !generated && !prefilled && !priority) {
    // identity order, completion only: copy the int32 column into the upper half of the
    // caller's int64 buffer, then widen in place front to back (element k is read from
    // byte 4N + 4k before byte 8k overwrites it)
    if (N) {
      int32_t* stage = reinterpret_cast<int32_t*>(completion_iter) + N;
      RS_CUDA(cudaMemcpy(stage, h.dev.comp, (size_t)N * 4, cudaMemcpyDeviceToHost));
      for (int k = 0; k < N; ++k) completion_iter[k] = stage[k];
    }
    return RS_OK;
  }
  std::vector<int> gen(generated ? N : 0), comp(completion_iter ? N : 0);
  std::vector<unsigned char> tab(h.rq_host.size());
  if (N && generated) RS_CUDA(cudaMemcpy(gen.data(), h.dev.gen, N * 4, cudaMemcpyDeviceToHost));
  if (N && completion_iter) RS_CUDA(cudaMemcpy(comp.data(), h.dev.comp, N * 4, cudaMemcpyDeviceToHost));
  if (prefilled || priority) RS_CUDA(cudaMemcpy(tab.data(), h.dev.rq_global, tab.size(), cudaMemcpyDeviceToHost));
  const RqView v = rq_carve(tab.data(), R);
  for (int a = 0; a < R; ++a) {
    const int lo = h.off[a], hi = h.off[a + 1];
    const int qa = (prefilled || priority) ? v.q[a] : 0;
    const double pa = priority ? v.prio[a] : 0.0;
    const bool ident = h.row_src.empty();
    for (int k = lo; k < hi; ++k) {
      const long long src = ident ? k : h.row_src[k];
      if (generated) generated[src] = gen[k];
      if (prefilled) prefilled[src] = (k - lo) < qa;
      if (completion_iter) completion_iter[src] = comp[k];
      if (priority) priority[src] = pa;
    }
  }
  return RS_OK;
}

int rs_engine_read_running(rs_engine* e, int32_t t, int32_t* rows, int32_t cap, int32_t* n_running) {
  if (!e || t < 0 || t >= (int)e->traces.size() || !n_running || cap < 0 || (cap > 0 && !rows))
    return fail(RS_EINVAL, "bad arguments");
  const HostTrace& h = e->traces[t];
  RS_CUDA(cudaSetDevice(e->device));
  if (e->ready) RS_CUDA(cudaEventSynchronize(e->ready));
  int n = 0;
  RS_CUDA(cudaMemcpy(&n, (const char*)h.dev.ctl + offsetof(Ctl, n_run), sizeof(int), cudaMemcpyDeviceToHost));
  *n_running = n;
  const int k = n < cap ? n : cap;
  if (k > 0) {
    std::vector<int> rr(k);
    RS_CUDA(cudaMemcpy(rr.data(), (const char*)h.dev.ctl + offsetof(Ctl, run_row), sizeof(int) * k,
                       cudaMemcpyDeviceToHost));
    for (int i = 0; i < k; ++i) rows[i] = (int32_t)(h.row_src.empty() ? rr[i] : h.row_src[rr[i]]);
  }
  return RS_OK;
}

int rs_engine_read_completion(rs_engine* e, int32_t t, int32_t* completion_iter) {
  if (!e || t < 0 || t >= (int)e->traces.size()) return fail(RS_EINVAL, "bad trace index");
  const HostTrace& h = e->traces[t];
  const int N = h.dev.N;
  RS_CUDA(cudaSetDevice(e->device));
  if (!N) return RS_OK;
  if (h.row_src.empty()) {  // admission order == trace order
    RS_CUDA(cudaMemcpy(completion_iter, h.dev.comp, (size_t)N * 4, cudaMemcpyDeviceToHost));
    return RS_OK;
  }
  std::vector<int> comp(N);
  RS_CUDA(cudaMemcpy(comp.data(), h.dev.comp, (size_t)N * 4, cudaMemcpyDeviceToHost));
  for (int k = 0; k < N; ++k) completion_iter[h.row_src[k]] = comp[k];
  return RS_OK;
}

void rs_engine_destroy(rs_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->done) {  // the last launch may still run on a non-blocking stream
    cudaEventSynchronize(e->done);
    cudaEventDestroy(e->done);
  }
  if (e->ready) {
    cudaEventSynchronize(e->ready);
    cudaEventDestroy(e->ready);
  }
  if (e->mbox) e->mbox_pooled ? cudaFreeAsync(e->mbox, 0) : cudaFree(e->mbox);
  if (e->d_peers) cudaFreeAsync(e->d_peers, 0);
  for (auto& h : e->traces) {
    for (void* p : h.allocs) cudaFree(p);
    if (h.arena_alloc) cudaFreeAsync(h.arena_alloc, 0);
    if (h.noise_buf) cudaFree(h.noise_buf);
  }
  if (e->d_traces) cudaFreeAsync(e->d_traces, 0);
  delete e;
}

int rs_device_clock_khz(int32_t device) {
  int khz = 0;
  if (cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device) != cudaSuccess) return 0;
  return khz;
}

int64_t rs_engine_device_bytes(const rs_engine* e) {
  if (!e) return 0;
  long long b = 0;
  for (auto& h : e->traces) b += h.bytes;
  return b;
}

int rs_pem_batch(int64_t n_sets, const int64_t* item_off, const int64_t* utok, const int32_t* remaining,
                 const uint8_t* prefilled, int64_t cap, int64_t mns, int64_t mnbt, const rs_cost_model* model,
                 double* values_out, int32_t device) {
  if (n_sets <= 0) return RS_OK;
  const long long n_items = item_off[n_sets];
  long long max_items = 1;
  for (long long s = 0; s < n_sets; ++s) max_items = std::max<long long>(max_items, item_off[s + 1] - item_off[s]);
  for (long long i = 0; i < n_items; ++i) {
    if (remaining[i] < 1) return fail(RS_EINVAL, "remainder items must have remaining >= 1");
    if (prefilled[i] && utok[i] != 0) return fail(RS_EINVAL, "prefilled items carry utok 0");
    if (utok[i] > cap) return fail(RS_EINFEASIBLE, "uncached tokens exceed cap");
  }
  RS_CUDA(cudaSetDevice(device));
  const int grid = (int)std::min<long long>(n_sets, 148 * 2);
  std::vector<unsigned char> segok(n_sets);
  for (long long s = 0; s < n_sets; ++s) {
    long long mx = 0;
    for (long long i = item_off[s]; i < item_off[s + 1]; ++i) mx = std::max<long long>(mx, utok[i]);
    segok[s] = mns * mx <= cap;
  }
  unsigned char* d_segok = nullptr;
  RS_CUDA(cudaMalloc(&d_segok, n_sets));
  RS_CUDA(cudaMemcpy(d_segok, segok.data(), n_sets, cudaMemcpyHostToDevice));
  RS_CUDA(cudaFuncSetAttribute(pem_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(UnitShared)));
  long long *d_off = nullptr, *d_utok = nullptr;
  int* d_rem = nullptr;
  unsigned char* d_pre = nullptr;
  double* d_out = nullptr;
  RS_CUDA(cudaMalloc(&d_off, (n_sets + 1) * 8));
  RS_CUDA(cudaMalloc(&d_utok, std::max<long long>(n_items, 1) * 8));
  RS_CUDA(cudaMalloc(&d_rem, std::max<long long>(n_items, 1) * 4));
  RS_CUDA(cudaMalloc(&d_pre, std::max<long long>(n_items, 1)));
  RS_CUDA(cudaMalloc(&d_out, n_sets * 8));
  RS_CUDA(cudaMemcpy(d_off, item_off, (n_sets + 1) * 8, cudaMemcpyHostToDevice));
  if (n_items) {
    RS_CUDA(cudaMemcpy(d_utok, utok, n_items * 8, cudaMemcpyHostToDevice));
    RS_CUDA(cudaMemcpy(d_rem, remaining, n_items * 4, cudaMemcpyHostToDevice));
    RS_CUDA(cudaMemcpy(d_pre, prefilled, n_items, cudaMemcpyHostToDevice));
  }
  PemModel m{model->alpha_p, model->beta_p, model->alpha_d, model->beta_d, cap, mns, mnbt};
  pem_batch_kernel<<<grid, kThreads, sizeof(UnitShared)>>>(n_sets, d_off, d_utok, d_rem, d_pre, d_segok, m, d_out);
  RS_CUDA(cudaGetLastError());
  RS_CUDA(cudaMemcpy(values_out, d_out, n_sets * 8, cudaMemcpyDeviceToHost));
  cudaFree(d_off);
  cudaFree(d_utok);
  cudaFree(d_rem);
  cudaFree(d_pre);
  cudaFree(d_out);
  cudaFree(d_segok);
  return RS_OK;
}

int rs_arrange(int32_t n_run, const int64_t* run_rel_id, const int64_t* run_output_limit, int64_t d_min_rel_id,
               int32_t n_prefill, int64_t prefill_utok, int64_t prefill_rel_id, int64_t prefill_output_limit,
               double m_plus, double m_minus, int64_t n_waiting, int32_t policy, const rs_cost_model* model,
               int32_t device, rs_iter_record* out) {
  if (n_run < 0 || n_run > kMaxRun || n_prefill < 0 || !model || !out) return fail(RS_EINVAL, "bad arranger input");
  if (policy < RS_POLICY_FCFS || policy > RS_POLICY_RELSERVE_DP) return fail(RS_EINVAL, "unknown policy");
  RS_CUDA(cudaSetDevice(device));
  long long* d = nullptr;
  rs_iter_record* d_out = nullptr;
  const size_t nb = std::max<int32_t>(n_run, 1) * sizeof(long long);
  RS_CUDA(cudaMalloc(&d, 3 * nb));
  RS_CUDA(cudaMalloc(&d_out, sizeof(rs_iter_record)));
  if (n_run) {
    RS_CUDA(cudaMemcpy(d, run_rel_id, n_run * sizeof(long long), cudaMemcpyHostToDevice));
    RS_CUDA(cudaMemcpy((char*)d + nb, run_output_limit, n_run * sizeof(long long), cudaMemcpyHostToDevice));
  }
  const int prefill_first = policy == RS_POLICY_FCFS || policy == RS_POLICY_SP;
  const int force = policy == RS_POLICY_RELSERVE_PP ? 1 : policy == RS_POLICY_RELSERVE_DP ? 2 : 0;
  arrange_kernel<<<1, 32>>>(n_run, d, (long long*)((char*)d + nb), d_min_rel_id, n_prefill, prefill_utok,
                            prefill_rel_id, prefill_output_limit, m_plus, m_minus, n_waiting, prefill_first, force,
                            *model, (long long*)((char*)d + 2 * nb), d_out);
  RS_CUDA(cudaGetLastError());
  RS_CUDA(cudaMemcpy(out, d_out, sizeof(rs_iter_record), cudaMemcpyDeviceToHost));
  cudaFree(d);
  cudaFree(d_out);
  return RS_OK;
}

int rs_waiting_argmin(const double* priority, const uint8_t* waiting, int64_t n, int32_t device, int64_t* head,
                      int64_t* count) {
  if (n < 0 || n > 0x7FFFFFF0LL || (n && (!priority || !waiting)) || !head || !count)
    return fail(RS_EINVAL, "bad waiting-order input");
  for (long long a = 0; a < n; ++a)  // okey orders every number; -0.0 would sort before +0.0
    if (waiting[a] && (priority[a] != priority[a] || (priority[a] == 0.0 && std::signbit(priority[a]))))
      return fail(RS_EINVAL, "priorities must be numbers (and not -0.0)");
  RS_CUDA(cudaSetDevice(device));
  double* d_p = nullptr;
  unsigned char* d_w = nullptr;
  long long* d_out = nullptr;
  const size_t m = (size_t)std::max<long long>(n, 1);
  RS_CUDA(cudaMalloc(&d_p, m * sizeof(double)));
  RS_CUDA(cudaMalloc(&d_w, m));
  RS_CUDA(cudaMalloc(&d_out, 2 * sizeof(long long)));
  if (n) {
    RS_CUDA(cudaMemcpy(d_p, priority, n * sizeof(double), cudaMemcpyHostToDevice));
    RS_CUDA(cudaMemcpy(d_w, waiting, n, cudaMemcpyHostToDevice));
  }
  waiting_argmin_kernel<<<1, kThreads>>>(n, d_p, d_w, d_out);
  RS_CUDA(cudaGetLastError());
  long long res[2];
  RS_CUDA(cudaMemcpy(res, d_out, sizeof res, cudaMemcpyDeviceToHost));
  cudaFree(d_p);
  cudaFree(d_w);
  cudaFree(d_out);
  *head = res[0];
  *count = res[1];
  return RS_OK;
}

int rs_choice_sequence(rs_pcg64_state* rng, int64_t n_calls, const int64_t* n, const int64_t* k, int64_t* idx_out,
                       int32_t device) {
  long long total = 0;
  for (long long c = 0; c < n_calls; ++c) {
    if (k[c] < 1 || k[c] >= n[c] || k[c] > kMaxSample || n[c] > 0xFFFFFFFFLL)
      return fail(RS_EINVAL, "choice call outside the replayed Floyd branch (1 <= k < n, k <= 64)");
    if (n[c] > 10000 && k[c] > n[c] / 50) return fail(RS_EUNSUPPORTED, "tail-shuffle branch");
    total += k[c];
  }
  RS_CUDA(cudaSetDevice(device));
  rs_pcg64_state* d_st = nullptr;
  long long *d_n = nullptr, *d_k = nullptr, *d_out = nullptr;
  RS_CUDA(cudaMalloc(&d_st, sizeof(rs_pcg64_state)));
  RS_CUDA(cudaMalloc(&d_n, std::max<long long>(n_calls, 1) * 8));
  RS_CUDA(cudaMalloc(&d_k, std::max<long long>(n_calls, 1) * 8));
  RS_CUDA(cudaMalloc(&d_out, std::max<long long>(total, 1) * 8));
  RS_CUDA(cudaMemcpy(d_st, rng, sizeof(rs_pcg64_state), cudaMemcpyHostToDevice));
  if (n_calls) {
    RS_CUDA(cudaMemcpy(d_n, n, n_calls * 8, cudaMemcpyHostToDevice));
    RS_CUDA(cudaMemcpy(d_k, k, n_calls * 8, cudaMemcpyHostToDevice));
  }
  choice_kernel<<<1, 32>>>(d_st, n_calls, d_n, d_k, d_out);
  RS_CUDA(cudaGetLastError());
  RS_CUDA(cudaMemcpy(rng, d_st, sizeof(rs_pcg64_state), cudaMemcpyDeviceToHost));
  if (total) RS_CUDA(cudaMemcpy(idx_out, d_out, total * 8, cudaMemcpyDeviceToHost));
  cudaFree(d_st);
  cudaFree(d_n);
  cudaFree(d_k);
  cudaFree(d_out);
  return RS_OK;
}

int rs_sort_pairs(const uint64_t* keys, const int32_t* values, int64_t n, uint64_t* keys_out, int32_t* values_out,
                  int32_t device) {
  if (n < 0 || (n && (!keys || !values || !keys_out || !values_out))) return fail(RS_EINVAL, "bad sort input");
  if (n > 0x7FFFFFF0LL) return fail(RS_EINVAL, "too many pairs");
  RS_CUDA(cudaSetDevice(device));
  if (n == 0) return RS_OK;
  DevBuf b;
  unsigned long long* k = nullptr;
  int* v = nullptr;
  RS_CUDA(b.get(&k, n));
  RS_CUDA(b.get(&v, n));
  RS_CUDA(cudaMemcpy(k, keys, n * 8, cudaMemcpyHostToDevice));
  RS_CUDA(cudaMemcpy(v, values, n * 4, cudaMemcpyHostToDevice));
  const int rc = sort_pairs_dev(k, v, n, 0);
  if (rc) return rc;
  RS_CUDA(cudaMemcpy(keys_out, k, n * 8, cudaMemcpyDeviceToHost));
  RS_CUDA(cudaMemcpy(values_out, v, n * 4, cudaMemcpyDeviceToHost));
  return RS_OK;
}

}  // extern "C"
