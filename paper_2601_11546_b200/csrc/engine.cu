// engine.cu -- the RelServe scheduler loop as one persistent sm_100a CTA per trace.
//
// Replaces the reference's per-iteration Python loops (Engine.run,
// pkg/src/relsim/engine.py:371-448).  Each CTA owns one trace and runs up to
// `max_iters` scheduler iterations per launch with no host round trip:
//
//   A  admission                      engine.py:243-269
//   B  Dynamic Priority Updater       priority.py:261-339 (reuse rule, numpy
//      PCG64 sample replay, utok*, block-cooperative PEM, starvation)
//   C  waiting-queue order: top-1     engine.py:277-281 (key (prio, arrival, rel_id)
//      by CTA argmin + waiting count  == (prio bits, admission rank))
//   D  candidates                     engine.py:285-308, arranger.py:71-112
//   E  decision + Delta projection    engine.py:387-416, arranger.py:115-179
//   F  state advance                  engine.py:315-363, 439-448, prefix-cache
//                                     LRU model (prefix_cache.py:65-138)
//
// Device state is a structure of arrays in HBM indexed by admission rank (the
// DPU's visit order); the per-trace control block (clock, queues, cache LRU
// bookkeeping, RNG) lives in shared memory during a launch.
//
// Only re-estimated relQueries are touched by the DPU: the reference's reuse
// rule (priority.py:261-266) makes every other value bit-identical to last
// iteration's, so the O(N) scans and write-backs of priority.py:266,307,309-312
// are replaced by per-relQuery state (prefilled prefix length q, done count).
//
// Prefix cache: for traces whose block trie is a forest of one shared chain
// per relQuery plus private per-row tails (checked on the host), the exact
// reference LRU (lazy heap over a global touch clock) reduces to: per
// relQuery the resident chain length m and the touch time c0 of its first
// block; per prefilled row a tail (start time, resident length) kept in a FIFO
// in insertion order; plus a small sorted list of tail-less resident chains.
// Eviction always takes the minimum-time unpinned leaf, which is either the
// FIFO head's deepest block or the first chain candidate's last block
// (see DESIGN.md "Prefix-cache model" for the argument).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/relserve.h"
#include "block.cuh"
#include "pcg64.cuh"
#include "pem.cuh"

namespace rsd {

constexpr int kMaxRun = 1024;      // device limit on max_num_seqs
constexpr int kMaxAct = 1024;      // partially-prefilled live relQueries
constexpr int kMaxCC = 256;        // tail-less resident chains
constexpr int kPemSmemItems = 1024;
constexpr int kWin = 768;          // FIFO window of the batched prefill eviction

struct FifoEnt {
  unsigned long long t0;  // touch time of the tail's first block
  int rank;               // owning relQuery
  int tres;               // resident blocks of the tail
};

struct CcEnt {
  unsigned long long key;  // touch time of the chain's last resident block
  int rank;
  int m;                   // resident chain blocks
};

// Persistent per-trace control block (global between launches, shared during one).
struct alignas(16) Ctl {
  double clock;
  long long iteration;
  long long kv;
  long long hit, miss;
  unsigned long long tclock;  // prefix-cache touch clock (prefix_cache.py:65-68)
  long long count;            // resident blocks
  long long n_log;
  long long fifo_head, fifo_tail;
  int n_admitted, live;
  int n_run, n_act;
  int status, error_detail;
  int cc_n, pad;
  rs_pcg64_state rng;
  long long phase[6];  // clock64 cycles per phase (+ scratch timestamp in [5])
  int run_row[kMaxRun];
  int run_rank[kMaxRun];
  int act[kMaxAct];
  int rrq[kMaxRun];  // relQueries with running rows (distinct)
  int n_rrq, pad2[3];
  CcEnt cc[kMaxCC];
};

static_assert(sizeof(Ctl) % 16 == 0, "Ctl is copied as int4");

struct TraceDev {
  int R, N, max_size, pad;
  const double* arrival;  // [R] by admission rank
  const int* row_off;     // [R+1]
  const int* ol;          // [R] output_limit
  const int* chain;       // [R] shared chain blocks P
  const long long* rel_id;
  const double* static_prio;
  const int* tok;  // [N] rank-ordered rows
  const int* out;
  double* prio;
  int* q;       // prefilled rows (always a prefix, SURVEY A-inv1)
  int* ndone;
  int* m;       // resident chain blocks
  unsigned long long* c0;
  int* ntails;  // rows of this relQuery with a resident tail
  int* nrun;    // running rows of this relQuery
  double* fps;
  double* lpe;
  double* lde;
  int* gen;
  int* comp;
  FifoEnt* fifo;
  long long fifo_cap;
  int* est;
  double* ratio;
  int* scr_cnt;   // [R] zeroed scratch: window tails per relQuery
  int* scr_last;  // [R] scratch (-1): last window index per relQuery
  void* pem_global;  // PemBuf backing for relQueries larger than kPemSmemItems
  rs_iter_record* log;
  long long log_cap;
  Ctl* ctl;
};

struct Params {
  const TraceDev* traces;
  rs_config cfg;
  rs_cost_model world;
  rs_cost_model pol;
  int use_dpu;
  int force;  // 0 none, 1 prefill (relserve-pp), 2 decode (relserve-dp)
  int prefill_first;
  int pad;
  long long max_iters;
};

struct Shared {
  Ctl c;
  PemShared pem;
  ArgminSmem am;
  ScanSmem scan;
  int go;
  int new_lo, new_hi;
  int head, W, taken;
  long long utok_sum;
  double m_plus, m_minus;
  int dmin_slot, n_est;
  int n_dist, act_dirty, rrq_dirty;
  int sorted_dist[kMaxRun];
  // batched prefill eviction
  int fp_bad, fp_ok, fp_popped, fp_win;
  long long fp_E;
  unsigned long long fp_c0_last;
  union {
    alignas(16) unsigned char pem_smem[pem_bytes_per_item() * kPemSmemItems + 16];
    struct {
      unsigned long long t0[kWin];
      unsigned long long c0[kWin];
      int rank[kWin];
      int tres[kWin];
      int mm[kWin];
      int last[kWin];  // 1 if this is the rank's last resident tail
    } win;
  };
};

__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7FF8000000000000LL); }

// ---------------------------------------------------------------------------
// Prefix-cache LRU model
//
// cc[] holds exactly the resident chains that have no resident tails (the
// only chain blocks that can be LRU leaves), sorted by the touch time of
// their last resident block.  An entry is removed as soon as its relQuery is
// prefilled again, so entries never go stale and carry their own length.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void cc_remove(Ctl& c, int rank) {
  for (int i = 0; i < c.cc_n; ++i)
    if (c.cc[i].rank == rank) {
      for (int j = i + 1; j < c.cc_n; ++j) c.cc[j - 1] = c.cc[j];
      c.cc_n--;
      return;
    }
}

__device__ __forceinline__ bool cc_insert(Ctl& c, unsigned long long key, int rank, int m) {
  if (c.cc_n == kMaxCC) return false;
  int pos = c.cc_n;
  while (pos > 0 && c.cc[pos - 1].key > key) {
    c.cc[pos] = c.cc[pos - 1];
    --pos;
  }
  c.cc[pos].key = key;
  c.cc[pos].rank = rank;
  c.cc[pos].m = m;
  c.cc_n++;
  return true;
}

// Evict the chain candidate at the front: k blocks from its end.
__device__ __forceinline__ void cc_evict_front(Ctl& c, const TraceDev& T, long long k) {
  CcEnt& e = c.cc[0];
  e.m -= (int)k;
  e.key -= (unsigned long long)k;
  T.m[e.rank] = e.m;
  c.count -= k;
  if (e.m == 0) {
    for (int i = 1; i < c.cc_n; ++i) c.cc[i - 1] = c.cc[i];
    c.cc_n--;
  }
}

// Exact per-row eviction (single thread): evict until count <= C.  cur_rank /
// cur_tail identify the pinned path (the row just inserted): its chain and,
// if it has one, its tail (the FIFO back).
__device__ int cache_evict(Ctl& c, const TraceDev& T, long long C, int cur_rank, bool cur_tail) {
  while (c.count > C) {
    const bool have_f = c.fifo_head < c.fifo_tail;
    unsigned long long kf = ~0ULL, kc = ~0ULL;
    FifoEnt fe;
    if (have_f) {
      fe = T.fifo[c.fifo_head % T.fifo_cap];
      kf = fe.t0 + (unsigned long long)(fe.tres - 1);
    }
    if (c.cc_n > 0) kc = c.cc[0].key;
    if (!have_f && c.cc_n == 0) return RS_ECACHE_PINNED;
    const long long need = c.count - C;
    if (kf < kc) {
      if (cur_tail && c.fifo_head == c.fifo_tail - 1) return RS_ECACHE_PINNED;
      const long long k = need < fe.tres ? need : fe.tres;
      fe.tres -= (int)k;
      c.count -= k;
      if (fe.tres == 0) {
        c.fifo_head++;
        const int a = fe.rank;
        const int nt = T.ntails[a] - 1;
        T.ntails[a] = nt;
        const int mm = T.m[a];
        if (nt == 0 && mm > 0 && !cc_insert(c, T.c0[a] + (unsigned long long)(mm - 1), a, mm))
          return RS_EUNSUPPORTED;
      } else {
        T.fifo[c.fifo_head % T.fifo_cap].tres = fe.tres;
      }
    } else {
      if (c.cc[0].rank == cur_rank) return RS_ECACHE_PINNED;
      const long long k = need < c.cc[0].m ? need : c.cc[0].m;
      cc_evict_front(c, T, k);
    }
  }
  return RS_OK;
}

// Exact path for one row: match_uncached(refresh=True, record=True) + insert
// (engine.py:321-323, prefix_cache.py:70-120).  Returns the row's uncached
// tokens, or -1 on error (status set).
__device__ long long prefill_row_cache(Ctl& c, const TraceDev& T, const Params& P, int a, int row) {
  const long long B = P.cfg.block_size;
  const int tok = T.tok[row];
  const int nb = (int)(tok / B);
  const int Pc = T.chain[a];
  const int T_len = nb - Pc;
  const int mb = T.m[a];
  const long long hit = B * mb;
  cc_remove(c, a);                                    // the chain is touched again
  c.hit += hit;
  c.miss += tok - hit;
  c.tclock += (unsigned long long)mb;                 // match touches the resident chain
  const unsigned long long c0 = c.tclock + 1;
  c.tclock += (unsigned long long)Pc;                 // insert touches the whole chain
  const unsigned long long t0 = c.tclock + 1;
  c.tclock += (unsigned long long)T_len;              // ... then the private tail
  c.count += (long long)(Pc - mb) + T_len;
  T.m[a] = Pc;
  T.c0[a] = c0;
  if (T_len > 0) {
    FifoEnt e;
    e.t0 = t0;
    e.rank = a;
    e.tres = T_len;
    T.fifo[c.fifo_tail % T.fifo_cap] = e;
    c.fifo_tail++;
    T.ntails[a] += 1;
  } else if (Pc > 0 && T.ntails[a] == 0) {
    if (!cc_insert(c, c0 + (unsigned long long)(Pc - 1), a, Pc)) {
      c.status = RS_EUNSUPPORTED;
      c.error_detail = 1;
      return -1;
    }
  }
  const int rc = cache_evict(c, T, P.cfg.capacity_blocks, a, T_len > 0);
  if (rc) {
    c.status = rc;
    c.error_detail = 2;
    return -1;
  }
  return tok - hit;
}


// Batched prefill advance (all threads).  All rows of a prefill batch belong
// to the head relQuery h, whose chain is pinned by every row's insert and is
// fully resident after the first one; if every row also has a private tail,
// the reference's per-row insert/evict interleaving evicts, in LRU order, the
// first E = max(0, count + new - C) blocks of the pre-batch resident set --
// whatever the interleaving, as long as E does not exceed those blocks.  So:
// per-row touch times and FIFO pushes by prefix sums, then one thread walks
// the FIFO head (staged in shared memory) and the chain candidates for E
// blocks.  Returns false (nothing changed) when the preconditions fail; the
// caller then runs the exact per-row path.
__device__ bool prefill_fast(const Params& P, const TraceDev& T, Shared& S, int h, int off, int q, int n,
                             long long& ut_out) {
  Ctl& c = S.c;
  const int tid = threadIdx.x;
  const long long B = P.cfg.block_size;
  const long long C = P.cfg.capacity_blocks;
  const int Pc = T.chain[h];
  const int m0 = T.m[h];
  const unsigned long long tc = c.tclock;
  const long long head0 = c.fifo_head, tail0 = c.fifo_tail, count0 = c.count;
  if (tid == 0) S.fp_bad = 0;
  __syncthreads();
  long long tokv[kMaxRun / kThreads], Tv[kMaxRun / kThreads], inclT[kMaxRun / kThreads];
  long long cT = 0, cTok = 0;
#pragma unroll
  for (int s = 0; s < kMaxRun / kThreads; ++s) {
    const int i = s * kThreads + tid;
    tokv[s] = 0;
    Tv[s] = 0;
    if (i < n) {
      tokv[s] = T.tok[off + q + i];
      Tv[s] = tokv[s] / B - Pc;
      if (Tv[s] <= 0) S.fp_bad = 1;
    }
    long long v[2] = {Tv[s], tokv[s]}, tot[2];
    block_incl_scan<2>(v, S.scan, tot);
    inclT[s] = cT + v[0];
    cT += tot[0];
    cTok += tot[1];
  }
  const long long newn = (long long)(Pc - m0) + cT;
  const long long E = count0 + newn > C ? count0 + newn - C : 0;
  const long long n_old = tail0 - head0;
  const int Wn = (int)(E < n_old ? E : n_old);
  if (S.fp_bad || E > count0 - m0 || Wn > kWin) return false;
  // FIFO pushes: row i's chain/tail touch times from prefix sums of touches
#pragma unroll
  for (int s = 0; s < kMaxRun / kThreads; ++s) {
    const int i = s * kThreads + tid;
    if (i < n) {
      const long long before = i == 0 ? 0 : (long long)m0 + (long long)(i - 1) * Pc + (long long)i * Pc + (inclT[s] - Tv[s]);
      const long long mb = i == 0 ? m0 : Pc;
      const unsigned long long c0i = tc + (unsigned long long)(before + mb + 1);
      FifoEnt e;
      e.t0 = c0i + (unsigned long long)Pc;
      e.rank = h;
      e.tres = (int)Tv[s];
      T.fifo[(tail0 + i) % T.fifo_cap] = e;
      if (i == n - 1) S.fp_c0_last = c0i;
    }
  }
  // stage the FIFO head (the oldest tails) and their relQueries' chain state
  for (int j = tid; j < Wn; j += kThreads) {
    const FifoEnt e = T.fifo[(head0 + j) % T.fifo_cap];
    S.win.t0[j] = e.t0;
    S.win.rank[j] = e.rank;
    S.win.tres[j] = e.tres;
    S.win.mm[j] = T.m[e.rank];
    S.win.c0[j] = T.c0[e.rank];
    atomicAdd(&T.scr_cnt[e.rank], 1);
    atomicMax(&T.scr_last[e.rank], j);
  }
  __syncthreads();
  for (int j = tid; j < Wn; j += kThreads) {
    const int a = S.win.rank[j];
    S.win.last[j] = (a != h && T.scr_last[a] == j && T.scr_cnt[a] == T.ntails[a]) ? 1 : 0;
  }
  __syncthreads();
  if (tid == 0) {
    cc_remove(c, h);
    long long need = E;
    int j = 0;
    bool ok = true;
    while (need > 0) {
      const unsigned long long kf = j < Wn ? S.win.t0[j] + (unsigned long long)(S.win.tres[j] - 1) : ~0ULL;
      const unsigned long long kc = c.cc_n > 0 ? c.cc[0].key : ~0ULL;
      if (kf == ~0ULL && kc == ~0ULL) {
        ok = false;
        break;
      }
      if (kf < kc) {
        const long long k = need < S.win.tres[j] ? need : S.win.tres[j];
        S.win.tres[j] -= (int)k;
        need -= k;
        c.count -= k;
        if (S.win.tres[j] == 0) {
          const int mm = S.win.mm[j];
          if (S.win.last[j] && mm > 0 &&
              !cc_insert(c, S.win.c0[j] + (unsigned long long)(mm - 1), S.win.rank[j], mm)) {
            ok = false;
            break;
          }
          ++j;
        }
      } else {
        const long long k = need < c.cc[0].m ? need : c.cc[0].m;
        need -= k;
        cc_evict_front(c, T, k);
      }
    }
    if (!ok) {
      c.status = RS_ECACHE_PINNED;
      c.error_detail = 4;
    }
    if (j < Wn) T.fifo[(head0 + j) % T.fifo_cap].tres = S.win.tres[j];
    S.fp_popped = j;
    const long long hitb = (long long)m0 + (long long)(n - 1) * Pc;
    c.hit += B * hitb;
    c.miss += cTok - B * hitb;
    ut_out = cTok - B * hitb;
    c.tclock = tc + (unsigned long long)(hitb + (long long)n * Pc + cT);
    c.count += newn;
    c.fifo_head = head0 + j;
    c.fifo_tail = tail0 + n;
    T.m[h] = Pc;
    T.c0[h] = S.fp_c0_last;
  }
  __syncthreads();
  const int popped = S.fp_popped;
  for (int j = tid; j < Wn; j += kThreads) {
    const int a = S.win.rank[j];
    if (j < popped) atomicSub(&T.ntails[a], 1);
    T.scr_cnt[a] = 0;
    T.scr_last[a] = -1;
  }
  if (tid == 0) atomicAdd(&T.ntails[h], n);
  __syncthreads();
  return true;
}

// ---------------------------------------------------------------------------
// DPU pieces
// ---------------------------------------------------------------------------

struct RqItems {  // remainder_items of one relQuery (priority.py:81-98)
  const int* tok;
  const int* out;
  const int* gen;
  int off, q, ol;
  double ratio;
  __device__ bool get(int i, long long& u, int& rem, int& pre) const {
    const int r = off + i;
    if (i < q) {
      const int g = gen[r];
      if (g >= out[r]) return false;  // done
      u = 0;
      rem = ol - g;
      pre = 1;
      return rem > 0;
    }
    const long long t = tok[r];
    // utok_approx: min(tok, floor(tok*ratio + 0.5)) (prefix_cache.py:172-176)
    const long long a = (long long)floor(__dadd_rn(__dmul_rn((double)t, ratio), 0.5));
    u = t < a ? t : a;
    rem = ol;
    pre = 0;
    return true;
  }
};

// sample_cache_miss_ratio (prefix_cache.py:141-169) for relQuery a; thread 0 only.
__device__ double sample_ratio(Pcg64& g, const TraceDev& T, const Params& P, int a) {
  const int off = T.row_off[a];
  const int size = T.row_off[a + 1] - off;
  const int q = T.q[a];
  const int n = size - q;  // unprefilled rows = [q, size) (A-inv1)
  if (n <= 0) return 0.0;
  const long long B = P.cfg.block_size;
  const long long mh = B * (long long)T.m[a];  // utok of an unprefilled row = tok - B*m
  const int k = (int)(P.cfg.sample_size < n ? P.cfg.sample_size : n);
  long long usum = 0, tsum = 0;
  if (k < n) {
    uint32_t idx[kMaxSample];
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

// thread 0 accumulates the cycles since the previous mark into phase k
__device__ __forceinline__ void phase_mark(Ctl& c, int k) {
  if (threadIdx.x == 0) {
    const long long now = clock64();
    c.phase[k] += now - c.phase[5];
    c.phase[5] = now;
  }
}

// ---------------------------------------------------------------------------
// One scheduler iteration.  Returns false when the trace stopped.
// ---------------------------------------------------------------------------

__device__ bool iterate(const Params& P, const TraceDev& T, Shared& S) {
  Ctl& c = S.c;
  const int tid = threadIdx.x;
  const rs_config& cfg = P.cfg;

  // ---- A: termination + admission (engine.py:375-380, 243-269)
  if (tid == 0) {
    S.go = 1;
    if (c.live == 0 && c.n_admitted == T.R) {
      c.status = RS_OK;
      S.go = 0;
    } else if (c.iteration >= cfg.iteration_limit) {
      c.status = RS_EABORT_LIMIT;
      S.go = 0;
    } else {
      int a = c.n_admitted;
      const int a0 = a;
      while (a < T.R && T.arrival[a] <= c.clock) {
        if (cfg.policy == RS_POLICY_SP) T.prio[a] = T.static_prio[a];
        else if (cfg.policy == RS_POLICY_FCFS) T.prio[a] = 0.0;
        ++a;
      }
      c.live += a - a0;
      c.n_admitted = a;
      S.new_lo = a0;
      S.new_hi = a;
    }
  }
  __syncthreads();
  if (!S.go) return false;
  phase_mark(c, 0);

  // ---- B: Dynamic Priority Updater (priority.py:287-339)
  if (P.use_dpu) {
    // re-estimated set, in visit (admission-rank) order: partially prefilled
    // live relQueries (sorted act list) then this iteration's arrivals
    const int n_act = c.n_act;
    const int n_new = S.new_hi - S.new_lo;
    const int n_est = n_act + n_new;
    if (tid == 0) {
      S.n_est = n_est;
      Pcg64 g = Pcg64::from(c.rng);
      for (int e = 0; e < n_est; ++e) {
        const int a = e < n_act ? c.act[e] : S.new_lo + (e - n_act);
        T.est[e] = a;
        T.ratio[e] = sample_ratio(g, T, P, a);
      }
      c.rng = g.to();
    }
    __syncthreads();
    PemModel pm;
    pm.ap = P.pol.alpha_p;
    pm.bp = P.pol.beta_p;
    pm.ad = P.pol.alpha_d;
    pm.bd = P.pol.beta_d;
    pm.cap = cfg.cap;
    pm.mns = cfg.max_num_seqs;
    pm.mnbt = cfg.max_num_batched_tokens;
    for (int e = 0; e < n_est; ++e) {
      const int a = T.est[e];
      RqItems it;
      it.tok = T.tok;
      it.out = T.out;
      it.gen = T.gen;
      it.off = T.row_off[a];
      it.q = T.q[a];
      it.ol = T.ol[a];
      it.ratio = T.ratio[e];
      const int n_src = T.row_off[a + 1] - it.off;
      PemBuf b = pem_carve(n_src <= kPemSmemItems ? (void*)S.pem_smem : T.pem_global,
                           n_src <= kPemSmemItems ? kPemSmemItems : T.max_size);
      const double v = block_pem(it, n_src, pm, b, S.pem);
      if (tid == 0) T.prio[a] = v;
    }
    // starvation override (priority.py:318-339): wholly-waiting = q == 0
    if (isfinite(cfg.tau)) {
      for (int a = tid; a < c.n_admitted; a += kThreads) {
        const int size = T.row_off[a + 1] - T.row_off[a];
        if (T.q[a] == 0 && size > 0) {
          const double uw = __ddiv_rn(__dsub_rn(c.clock, T.arrival[a]), (double)size);
          if (uw > cfg.tau) T.prio[a] = 0.0;
        }
      }
    }
    __syncthreads();
  } else if (tid == 0) {
    S.n_est = 0;
  }
  phase_mark(c, 1);

  // ---- C: waiting head = argmin (prio, rank) over relQueries with pending rows
  {
    unsigned long long key = ~0ULL;
    long long idx = 0x7FFFFFFFFFFFFFFFLL;
    long long w = 0;
    for (int a = tid; a < c.n_admitted; a += kThreads) {
      const int size = T.row_off[a + 1] - T.row_off[a];
      if (T.q[a] < size) {
        ++w;
        argmin_merge(key, idx, dbits(T.prio[a]), a);
      }
    }
    const long long W = block_sum(w, S.scan);
    block_argmin(key, idx, S.am);
    if (tid == 0) {
      S.W = (int)W;
      S.head = W > 0 ? (int)idx : -1;
    }
  }
  phase_mark(c, 2);

  // ---- D: candidates (engine.py:285-308)
  {
    // decode candidate = running list; m+ and the first running row attaining it
    unsigned long long key = ~0ULL;
    long long idx = 0x7FFFFFFFFFFFFFFFLL;
    for (int j = tid; j < c.n_run; j += kThreads) argmin_merge(key, idx, dbits(T.prio[c.run_rank[j]]), j);
    block_argmin(key, idx, S.am);
    if (tid == 0) {
      S.dmin_slot = c.n_run > 0 ? (int)idx : -1;
      S.m_plus = c.n_run > 0 ? T.prio[c.run_rank[idx]] : qnan();
    }
    // prefill candidate: leading run of the head's pending rows (arranger.py:80-112)
    const int h = S.head;
    int J = 0, off = 0, q = 0;
    long long B = cfg.block_size, mh = 0, olh = 0;
    if (h >= 0) {
      off = T.row_off[h];
      q = T.q[h];
      const int pend = T.row_off[h + 1] - off - q;
      const long long room = cfg.max_num_seqs - c.n_run;
      J = room <= 0 ? 0 : (int)(pend < room ? pend : room);
      mh = B * (long long)T.m[h];
      olh = T.ol[h];
    }
    const long long headroom = cfg.cap - c.kv;
    long long cu = 0, ck = 0;
    long long first_bad = J;
    for (int base = 0; base < J; base += kThreads) {
      const int j = base + tid;
      long long v[2] = {0, 0};
      if (j < J) {
        const long long t = T.tok[off + q + j];
        v[0] = t - mh;   // exact utok (match_uncached, refresh=False)
        v[1] = t + olh;  // kv need
      }
      long long tot[2];
      block_incl_scan<2>(v, S.scan, tot);
      long long bad = 0x7FFFFFFFFFFFFFFFLL;
      if (j < J) {
        const long long U = cu + v[0], K = ck + v[1];
        if ((j > 0 && U > cfg.max_num_batched_tokens) || K > headroom) bad = j;
      }
      unsigned long long kk = (unsigned long long)bad;
      long long ii = bad;
      block_argmin(kk, ii, S.am);
      if ((long long)kk < first_bad) first_bad = (long long)kk;
      cu += tot[0];
      ck += tot[1];
      if (first_bad < J) break;
    }
    if (tid == 0) S.taken = (int)first_bad;
    __syncthreads();
    // utok sum of the taken rows
    long long us = 0;
    for (int j = tid; j < S.taken; j += kThreads) us += T.tok[off + q + j] - mh;
    us = block_sum(us, S.scan);
    if (tid == 0) {
      S.utok_sum = us;
      S.m_minus = S.taken > 0 ? T.prio[h] : qnan();
    }
    __syncthreads();
  }

  // ---- E: decision (engine.py:387-433, arranger.py:115-179)
  const bool has_p = S.taken > 0, has_d = c.n_run > 0;
  bool need_proj = false;
  if (!P.prefill_first && has_p && has_d && S.m_plus <= S.m_minus) need_proj = true;
  if (need_proj) {
    // distinct running relQueries (the rrq list), sorted by rel_id (engine.py:406-408)
    const int nd = c.n_rrq;
    for (int i = tid; i < nd; i += kThreads) {
      const long long ri = T.rel_id[c.rrq[i]];
      int pos = 0;
      for (int k = 0; k < nd; ++k) pos += T.rel_id[c.rrq[k]] < ri;
      S.sorted_dist[pos] = c.rrq[i];
    }
    if (tid == 0) S.n_dist = nd;
    __syncthreads();
  }
  if (tid == 0) {
    int action, kase;
    double dp = qnan(), dm = qnan(), dt = qnan();
    double mp = S.m_plus, mmn = S.m_minus;
    if (P.prefill_first) {
      kase = RS_CASE_FORCED;
      if (has_p) action = RS_ACTION_PREFILL;
      else if (has_d) action = RS_ACTION_DECODE;
      else {
        action = RS_ACTION_IDLE;
        mp = mmn = qnan();
      }
    } else {
      double ddp = 0, ddm = 0, ddt = 0;
      if (need_proj) {  // project_delta (arranger.py:115-143), left-to-right fp64
        const rs_cost_model& m = P.pol;
        const double l_prefill = __dadd_rn(__dmul_rn(m.alpha_p, (double)S.utok_sum), m.beta_p);
        const long long ol_p = T.ol[S.head];
        ddp = __dmul_rn(l_prefill, (double)S.n_dist);
        long long max_ol = 0;
        const double adn = __dmul_rn(m.alpha_d, (double)S.taken);
        for (int i = 0; i < S.n_dist; ++i) {
          const long long ol = T.ol[S.sorted_dist[i]];
          const long long mn = ol < ol_p ? ol : ol_p;
          ddp = __dadd_rn(ddp, __dmul_rn(adn, (double)mn));
          max_ol = ol > max_ol ? ol : max_ol;
        }
        const long long mn = ol_p < max_ol ? ol_p : max_ol;
        ddm = -__dmul_rn(__dmul_rn((double)S.W, m.beta_d), (double)mn);
        ddt = __dadd_rn(ddp, ddm);
      }
      if (!has_p && !has_d) {
        action = RS_ACTION_IDLE;
        kase = RS_CASE_FORCED;
        mp = mmn = qnan();
      } else if (!has_d) {
        action = RS_ACTION_PREFILL;
        kase = RS_CASE_FORCED;
      } else if (!has_p) {
        action = RS_ACTION_DECODE;
        kase = RS_CASE_FORCED;
      } else if (c.run_rank[S.dmin_slot] == S.head) {
        action = RS_ACTION_PREFILL;
        kase = RS_CASE_INTERNAL;
      } else if (S.m_plus > S.m_minus) {
        action = RS_ACTION_PREFILL;
        kase = RS_CASE_PREEMPT;
      } else {
        kase = RS_CASE_TRANSITIONAL;
        dp = ddp;
        dm = ddm;
        dt = ddt;
        if (P.force == 1) action = RS_ACTION_PREFILL;
        else if (P.force == 2) action = RS_ACTION_DECODE;
        else action = (ddt < 0) ? RS_ACTION_PREFILL : RS_ACTION_DECODE;
      }
    }
    S.go = action;  // reuse as the action slot
    if (cfg.log_decisions && T.log_cap > 0) {
      rs_iter_record& r = T.log[c.n_log % T.log_cap];
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
  __syncthreads();
  const int action = S.go;
  phase_mark(c, 3);

  // ---- F: execute
  if (action == RS_ACTION_PREFILL) {  // _execute_prefill (engine.py:315-341)
    const int h = S.head;
    const int off = T.row_off[h];
    const int q = T.q[h];
    const int n = S.taken;
    const int n_run0 = c.n_run;
    long long ut = 0;
    const bool fast = prefill_fast(P, T, S, h, off, q, n, ut);
    if (tid == 0) {
      bool ok = c.status == RS_RUNNING;
      if (!fast && ok) {
        for (int i = 0; i < n; ++i) {
          const long long u = prefill_row_cache(c, T, P, h, off + q + i);
          if (u < 0) {
            ok = false;
            break;
          }
          ut += u;
        }
      }
      if (ok) {
        const double start = c.clock;
        const double dur = __dadd_rn(__dmul_rn(P.world.alpha_p, (double)ut), P.world.beta_p);
        c.n_run = n_run0 + n;
        T.q[h] = q + n;
        if (T.nrun[h] == 0) c.rrq[c.n_rrq++] = h;
        T.nrun[h] += n;
        if (q == 0 && P.use_dpu) {  // becomes partially prefilled: join the re-estimate list
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
        if (isnan(T.fps[h])) T.fps[h] = start;
        T.lpe[h] = c.clock;
        if (cfg.log_decisions && T.log_cap > 0) {
          rs_iter_record& r = T.log[c.n_log % T.log_cap];
          r.batch_rq = h;
          r.batch_first = q;
          r.batch_n = n;
        }
      }
      S.go = ok && c.status == RS_RUNNING;
    }
    // running list append + kv reservation (engine.py:326-329)
    long long kv = 0;
    const int ol = T.ol[h];
    for (int i = tid; i < n; i += kThreads) {
      c.run_row[n_run0 + i] = off + q + i;
      c.run_rank[n_run0 + i] = h;
      kv += (long long)T.tok[off + q + i] + ol;
    }
    kv = block_sum(kv, S.scan);
    if (tid == 0) c.kv += kv;
    __syncthreads();
    if (!S.go) return false;
  } else if (action == RS_ACTION_DECODE) {  // _execute_decode (engine.py:343-363)
    const int n = c.n_run;
    double clk = 0;
    if (tid == 0) {
      S.act_dirty = 0;
      S.rrq_dirty = 0;
    }
    __syncthreads();
    clk = __dadd_rn(c.clock, __dadd_rn(__dmul_rn(P.world.alpha_d, (double)n), P.world.beta_d));
    long long kv_free = 0;
    int keep_flag[kMaxRun / kThreads];
#pragma unroll
    for (int s = 0; s < kMaxRun / kThreads; ++s) {
      const int j = s * kThreads + tid;
      keep_flag[s] = 0;
      if (j < n) {
        const int r = c.run_row[j];
        const int a = c.run_rank[j];
        const int g = T.gen[r] + 1;
        T.gen[r] = g;
        if (g >= T.out[r]) {
          T.comp[r] = (int)c.iteration;
          if (atomicSub(&T.nrun[a], 1) == 1) S.rrq_dirty = 1;
          kv_free += (long long)T.tok[r] + T.ol[a];
          const int size = T.row_off[a + 1] - T.row_off[a];
          if (atomicAdd(&T.ndone[a], 1) + 1 == size) {
            T.lde[a] = clk;
            atomicSub(&c.live, 1);
            S.act_dirty = 1;
          }
        } else {
          keep_flag[s] = 1;
        }
      }
    }
    kv_free = block_sum(kv_free, S.scan);
    // stable compaction of the running list
    int cbase = 0;
    int new_row[kMaxRun / kThreads], new_rank[kMaxRun / kThreads];
#pragma unroll
    for (int s = 0; s < kMaxRun / kThreads; ++s) {
      const int j = s * kThreads + tid;
      new_row[s] = j < n ? c.run_row[j] : 0;
      new_rank[s] = j < n ? c.run_rank[j] : 0;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kMaxRun / kThreads; ++s) {
      long long v[1] = {keep_flag[s]};
      long long tot[1];
      block_incl_scan<1>(v, S.scan, tot);
      if (keep_flag[s]) {
        c.run_row[cbase + v[0] - 1] = new_row[s];
        c.run_rank[cbase + v[0] - 1] = new_rank[s];
      }
      cbase += (int)tot[0];
    }
    __syncthreads();
    if (tid == 0) {
      c.n_run = cbase;
      c.kv -= kv_free;
      c.clock = clk;
      if (cfg.log_decisions && T.log_cap > 0) T.log[c.n_log % T.log_cap].batch_n = n;
      if (S.rrq_dirty) {
        int w = 0;
        for (int i = 0; i < c.n_rrq; ++i)
          if (T.nrun[c.rrq[i]] > 0) c.rrq[w++] = c.rrq[i];
        c.n_rrq = w;
      }
      if (S.act_dirty && P.use_dpu) {  // drop retired relQueries from the re-estimate list
        int w = 0;
        for (int i = 0; i < c.n_act; ++i) {
          const int a = c.act[i];
          if (T.ndone[a] < T.row_off[a + 1] - T.row_off[a]) c.act[w++] = a;
        }
        c.n_act = w;
      }
    }
  } else {  // idle (engine.py:439-447)
    if (tid == 0) {
      if (c.n_admitted >= T.R) {
        c.status = c.live ? RS_EABORT_IDLE : RS_OK;
        S.go = 0;
        if (cfg.log_decisions && T.log_cap > 0) {
          T.log[c.n_log % T.log_cap].kv_reserved = c.kv;
          c.n_log++;
        }
      } else {
        const double nxt = T.arrival[c.n_admitted];
        if (nxt > c.clock) c.clock = nxt;
        S.go = 1;
      }
    }
    __syncthreads();
    if (!S.go) return false;
  }
  if (tid == 0) {
    if (cfg.log_decisions && T.log_cap > 0) {
      T.log[c.n_log % T.log_cap].kv_reserved = c.kv;
      c.n_log++;
    }
    c.iteration++;
  }
  phase_mark(c, 4);
  __syncthreads();
  return true;
}

__global__ void __launch_bounds__(kThreads, 1) engine_kernel(Params P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Shared& S = *reinterpret_cast<Shared*>(smem_raw);
  const TraceDev& T = P.traces[blockIdx.x];
  {
    const int4* src = reinterpret_cast<const int4*>(T.ctl);
    int4* dst = reinterpret_cast<int4*>(&S.c);
    for (int i = threadIdx.x; i < (int)(sizeof(Ctl) / 16); i += kThreads) dst[i] = src[i];
  }
  __syncthreads();
  if (S.c.status != RS_RUNNING) return;
  if (threadIdx.x == 0) S.c.phase[5] = clock64();
  for (long long it = 0; it < P.max_iters; ++it)
    if (!iterate(P, T, S)) break;
  __syncthreads();
  {
    const int4* src = reinterpret_cast<const int4*>(&S.c);
    int4* dst = reinterpret_cast<int4*>(T.ctl);
    for (int i = threadIdx.x; i < (int)(sizeof(Ctl) / 16); i += kThreads) dst[i] = src[i];
  }
}

// ---------------------------------------------------------------------------
// Unit kernels
// ---------------------------------------------------------------------------

struct ArrItems {
  const long long* utok;
  const int* rem;
  const unsigned char* pre;
  long long off;
  __device__ bool get(int i, long long& u, int& r, int& p) const {
    u = utok[off + i];
    r = rem[off + i];
    p = pre[off + i];
    return true;
  }
};

struct PemBatchShared {
  PemShared pem;
};

__global__ void __launch_bounds__(kThreads, 1)
    pem_batch_kernel(long long n_sets, const long long* item_off, const long long* utok, const int* rem,
                     const unsigned char* pre, PemModel m, void* scratch, int scratch_items, double* out) {
  __shared__ PemBatchShared S;
  PemBuf b = pem_carve((char*)scratch + (size_t)blockIdx.x * pem_buf_size(scratch_items), scratch_items);
  for (long long s = blockIdx.x; s < n_sets; s += gridDim.x) {
    ArrItems it{utok, rem, pre, item_off[s]};
    const double v = block_pem(it, (int)(item_off[s + 1] - item_off[s]), m, b, S.pem);
    if (threadIdx.x == 0) out[s] = v;
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

#define RS_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess) return fail(RS_ECUDA, std::string(#call ": ") + cudaGetErrorString(_e)); \
  } while (0)

struct HostTrace {
  TraceDev dev{};
  std::vector<int> rank_of;     // trace index -> rank
  std::vector<int> order;       // rank -> trace index
  std::vector<long long> row_src;  // rank-ordered row -> trace-order row
  std::vector<void*> allocs;
  long long bytes = 0;
  long long log_read = 0;
};

template <typename T>
int dalloc(HostTrace& h, T** p, size_t n, const void* src = nullptr, int fill_byte = -1) {
  if (n == 0) n = 1;
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, n * sizeof(T));
  if (e != cudaSuccess) return fail(RS_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  h.allocs.push_back(q);
  h.bytes += (long long)(n * sizeof(T));
  if (src) {
    e = cudaMemcpy(q, src, n * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(RS_ECUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
  } else if (fill_byte >= 0) {
    e = cudaMemset(q, fill_byte, n * sizeof(T));
    if (e != cudaSuccess) return fail(RS_ECUDA, std::string("cudaMemset: ") + cudaGetErrorString(e));
  }
  *p = (T*)q;
  return RS_OK;
}

}  // namespace

struct rs_engine {
  int device = 0;
  Params params{};
  std::vector<HostTrace> traces;
  TraceDev* d_traces = nullptr;
  size_t smem = 0;
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
  if (cfg->noise_sigma > 0) return fail(RS_EUNSUPPORTED, "world-model noise is not on the device path");
  if (dpu && cfg->sample_size < 1) return fail(RS_EINVAL, "sample_size must be positive");
  if (dpu && cfg->sample_size > kMaxSample)
    return fail(RS_EUNSUPPORTED, "sample_size above the device limit (64)");
  if (cfg->max_num_seqs > kMaxRun) return fail(RS_EUNSUPPORTED, "max_num_seqs above the device limit (1024)");
  return RS_OK;
}

static int build_trace(const rs_trace_view& v, const rs_config* cfg, const rs_pcg64_state& rng,
                       long long log_cap, HostTrace& h) {
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
  std::vector<int> tok(N), out(N);
  h.row_src.resize(N);
  int max_size = 1;
  long long max_nb = 0;
  long long k = 0;
  off[0] = 0;
  for (long long a = 0; a < R; ++a) {
    const int t = h.order[a];
    arrival[a] = v.arrival[t];
    ol[a] = v.output_limit[t];
    chain[a] = v.chain_blocks ? v.chain_blocks[t] : 0;
    relid[a] = v.rel_id[t];
    if (v.static_prio) sprio[a] = v.static_prio[t];
    const long long lo = v.row_off[t], hi = v.row_off[t + 1];
    if (hi < lo) return fail(RS_EINVAL, "row_off must be non-decreasing");
    if (ol[a] <= 0) return fail(RS_EINVAL, "output_limit must be positive");
    if (hi - lo > max_size) max_size = (int)(hi - lo);
    if (dpu && cfg->sample_size > 200 && hi - lo > 10000)
      return fail(RS_EUNSUPPORTED, "Generator.choice tail-shuffle branch is not replayed");
    for (long long r = lo; r < hi; ++r) {
      tok[k] = v.tok[r];
      out[k] = v.out[r];
      h.row_src[k] = r;
      if (tok[k] <= 0) return fail(RS_EINVAL, "request tokens must be non-empty");
      if (out[k] < 1 || out[k] > ol[a]) return fail(RS_EINVAL, "actual_output_len out of range");
      if ((long long)tok[k] + ol[a] > cfg->cap) {
        char msg[200];
        snprintf(msg, sizeof msg, "request %lld/%lld needs %lld KV tokens > cap %lld", (long long)relid[a],
                 (long long)(r - lo), (long long)tok[k] + ol[a], (long long)cfg->cap);
        return fail(RS_EINFEASIBLE, msg);
      }
      const long long nb = tok[k] / cfg->block_size;
      if (nb < chain[a]) return fail(RS_EUNSUPPORTED, "chain_blocks exceeds a row's whole blocks");
      if (nb > max_nb) max_nb = nb;
      ++k;
    }
    off[a + 1] = (int)k;
  }
  if (max_nb > cfg->capacity_blocks)
    return fail(RS_EUNSUPPORTED, "a request has more whole blocks than the cache capacity (truncated insert)");
  TraceDev& d = h.dev;
  d.R = (int)R;
  d.N = (int)N;
  d.max_size = max_size;
  int rc;
#define TRY(x) \
  if ((rc = (x))) return rc
  TRY(dalloc(h, (double**)&d.arrival, R, arrival.data()));
  TRY(dalloc(h, (int**)&d.row_off, R + 1, off.data()));
  TRY(dalloc(h, (int**)&d.ol, R, ol.data()));
  TRY(dalloc(h, (int**)&d.chain, R, chain.data()));
  TRY(dalloc(h, (long long**)&d.rel_id, R, relid.data()));
  TRY(dalloc(h, (double**)&d.static_prio, R, sprio.data()));
  TRY(dalloc(h, (int**)&d.tok, N, tok.data()));
  TRY(dalloc(h, (int**)&d.out, N, out.data()));
  TRY(dalloc(h, &d.prio, R, nullptr, 0));
  TRY(dalloc(h, &d.q, R, nullptr, 0));
  TRY(dalloc(h, &d.ndone, R, nullptr, 0));
  TRY(dalloc(h, &d.m, R, nullptr, 0));
  TRY(dalloc(h, &d.c0, R, nullptr, 0));
  TRY(dalloc(h, &d.ntails, R, nullptr, 0));
  TRY(dalloc(h, &d.nrun, R, nullptr, 0));
  std::vector<double> nanv(R, NAN);
  TRY(dalloc(h, &d.fps, R, nanv.data()));
  TRY(dalloc(h, &d.lpe, R, nanv.data()));
  TRY(dalloc(h, &d.lde, R, nanv.data()));
  TRY(dalloc(h, &d.gen, N, nullptr, 0));
  TRY(dalloc(h, &d.comp, N, nullptr, 0xFF));
  d.fifo_cap = cfg->capacity_blocks + kMaxRun + 2;  // batched pushes precede evictions
  TRY(dalloc(h, &d.fifo, d.fifo_cap, nullptr, 0));
  TRY(dalloc(h, &d.est, R + kMaxAct, nullptr, 0));
  TRY(dalloc(h, &d.ratio, R + kMaxAct, nullptr, 0));
  TRY(dalloc(h, &d.scr_cnt, R, nullptr, 0));
  TRY(dalloc(h, &d.scr_last, R, nullptr, 0xFF));
  if (max_size > kPemSmemItems) {
    TRY(dalloc(h, (unsigned char**)&d.pem_global, pem_buf_size(max_size), nullptr, 0));
  }
  d.log_cap = log_cap;
  if (log_cap > 0) TRY(dalloc(h, &d.log, log_cap, nullptr, 0));
  Ctl* ctl = (Ctl*)calloc(1, sizeof(Ctl));
  if (!ctl) return fail(RS_ENOMEM, "host alloc");
  ctl->status = RS_RUNNING;
  ctl->rng = rng;
  rc = dalloc(h, &d.ctl, 1, ctl);
  free(ctl);
  if (rc) return rc;
#undef TRY
  return RS_OK;
}

int rs_engine_create(const rs_trace_view* traces, int32_t n_traces, const rs_config* cfg,
                     const rs_cost_model* world, const rs_cost_model* policy_model,
                     const rs_pcg64_state* rng, int32_t device, int64_t log_capacity, rs_engine** out) {
  *out = nullptr;
  if (n_traces <= 0) return fail(RS_EINVAL, "n_traces must be positive");
  int rc = validate_config(cfg);
  if (rc) return rc;
  RS_CUDA(cudaSetDevice(device));
  rs_engine* e = new rs_engine();
  e->device = device;
  e->traces.resize(n_traces);
  for (int t = 0; t < n_traces; ++t) {
    rc = build_trace(traces[t], cfg, rng[t], log_capacity, e->traces[t]);
    if (rc) {
      std::string keep = g_err;
      rs_engine_destroy(e);
      g_err = keep;
      return rc;
    }
  }
  std::vector<TraceDev> devs(n_traces);
  for (int t = 0; t < n_traces; ++t) devs[t] = e->traces[t].dev;
  if (cudaMalloc(&e->d_traces, sizeof(TraceDev) * n_traces) != cudaSuccess ||
      cudaMemcpy(e->d_traces, devs.data(), sizeof(TraceDev) * n_traces, cudaMemcpyHostToDevice) != cudaSuccess) {
    rs_engine_destroy(e);
    return fail(RS_ECUDA, "trace table upload failed");
  }
  Params& p = e->params;
  p.traces = e->d_traces;
  p.cfg = *cfg;
  p.world = *world;
  p.pol = *policy_model;
  p.use_dpu = cfg->policy >= RS_POLICY_RELSERVE;
  p.force = cfg->policy == RS_POLICY_RELSERVE_PP ? 1 : cfg->policy == RS_POLICY_RELSERVE_DP ? 2 : 0;
  p.prefill_first = cfg->policy == RS_POLICY_FCFS || cfg->policy == RS_POLICY_SP;
  e->smem = sizeof(Shared);
  cudaError_t ce = cudaFuncSetAttribute(engine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e->smem);
  if (ce != cudaSuccess) {
    rs_engine_destroy(e);
    return fail(RS_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(ce));
  }
  *out = e;
  return RS_OK;
}

int rs_engine_step(rs_engine* e, int64_t max_iters, void* stream) {
  if (!e) return fail(RS_EINVAL, "null engine");
  RS_CUDA(cudaSetDevice(e->device));
  long long cap = e->params.cfg.log_decisions ? e->traces[0].dev.log_cap : max_iters;
  if (e->params.cfg.log_decisions && cap > 0 && max_iters > cap) max_iters = cap;
  Params p = e->params;
  p.max_iters = max_iters;
  engine_kernel<<<(unsigned)e->traces.size(), kThreads, e->smem, (cudaStream_t)stream>>>(p);
  RS_CUDA(cudaGetLastError());
  return RS_OK;
}

int rs_engine_status(rs_engine* e, void* stream, rs_trace_status* st) {
  if (!e) return fail(RS_EINVAL, "null engine");
  RS_CUDA(cudaSetDevice(e->device));
  RS_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  const size_t head = offsetof(Ctl, run_row);
  std::vector<unsigned char> buf(head);
  for (size_t t = 0; t < e->traces.size(); ++t) {
    RS_CUDA(cudaMemcpy(buf.data(), e->traces[t].dev.ctl, head, cudaMemcpyDeviceToHost));
    const Ctl* c = reinterpret_cast<const Ctl*>(buf.data());
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
    for (int k = 0; k < 5; ++k) s.phase_cycles[k] = c->phase[k];
  }
  return RS_OK;
}

int rs_engine_read_log(rs_engine* e, int32_t t, int64_t first, int64_t count, rs_iter_record* out) {
  if (!e || t < 0 || t >= (int)e->traces.size()) return fail(RS_EINVAL, "bad trace index");
  const TraceDev& d = e->traces[t].dev;
  if (count <= 0) return RS_OK;
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

int rs_engine_read_ledgers(rs_engine* e, int32_t t, double* arrival, double* fps, double* lpe, double* lde) {
  if (!e || t < 0 || t >= (int)e->traces.size()) return fail(RS_EINVAL, "bad trace index");
  const HostTrace& h = e->traces[t];
  const int R = h.dev.R;
  RS_CUDA(cudaSetDevice(e->device));
  std::vector<double> a(R), b(R), c(R), d(R);
  if (R) {
    RS_CUDA(cudaMemcpy(a.data(), h.dev.arrival, R * 8, cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(b.data(), h.dev.fps, R * 8, cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(c.data(), h.dev.lpe, R * 8, cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(d.data(), h.dev.lde, R * 8, cudaMemcpyDeviceToHost));
  }
  for (int r = 0; r < R; ++r) {
    const int i = h.order[r];
    if (arrival) arrival[i] = a[r];
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
  std::vector<int> gen(N), comp(N), q(R), off(R + 1);
  std::vector<double> prio(R);
  if (N) {
    RS_CUDA(cudaMemcpy(gen.data(), h.dev.gen, N * 4, cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(comp.data(), h.dev.comp, N * 4, cudaMemcpyDeviceToHost));
  }
  if (R) {
    RS_CUDA(cudaMemcpy(q.data(), h.dev.q, R * 4, cudaMemcpyDeviceToHost));
    RS_CUDA(cudaMemcpy(prio.data(), h.dev.prio, R * 8, cudaMemcpyDeviceToHost));
  }
  RS_CUDA(cudaMemcpy(off.data(), h.dev.row_off, (R + 1) * 4, cudaMemcpyDeviceToHost));
  for (int a = 0; a < R; ++a) {
    for (int k = off[a]; k < off[a + 1]; ++k) {
      const long long src = h.row_src[k];
      if (generated) generated[src] = gen[k];
      if (prefilled) prefilled[src] = (k - off[a]) < q[a];
      if (completion_iter) completion_iter[src] = comp[k];
      if (priority) priority[src] = prio[a];
    }
  }
  return RS_OK;
}

void rs_engine_destroy(rs_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  for (auto& h : e->traces)
    for (void* p : h.allocs) cudaFree(p);
  if (e->d_traces) cudaFree(e->d_traces);
  delete e;
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
  const int grid = (int)std::min<long long>(n_sets, 148);
  long long *d_off = nullptr, *d_utok = nullptr;
  int* d_rem = nullptr;
  unsigned char *d_pre = nullptr, *d_scr = nullptr;
  double* d_out = nullptr;
  const size_t scr = pem_buf_size((int)max_items) * grid;
  RS_CUDA(cudaMalloc(&d_off, (n_sets + 1) * 8));
  RS_CUDA(cudaMalloc(&d_utok, std::max<long long>(n_items, 1) * 8));
  RS_CUDA(cudaMalloc(&d_rem, std::max<long long>(n_items, 1) * 4));
  RS_CUDA(cudaMalloc(&d_pre, std::max<long long>(n_items, 1)));
  RS_CUDA(cudaMalloc(&d_scr, scr));
  RS_CUDA(cudaMalloc(&d_out, n_sets * 8));
  RS_CUDA(cudaMemcpy(d_off, item_off, (n_sets + 1) * 8, cudaMemcpyHostToDevice));
  if (n_items) {
    RS_CUDA(cudaMemcpy(d_utok, utok, n_items * 8, cudaMemcpyHostToDevice));
    RS_CUDA(cudaMemcpy(d_rem, remaining, n_items * 4, cudaMemcpyHostToDevice));
    RS_CUDA(cudaMemcpy(d_pre, prefilled, n_items, cudaMemcpyHostToDevice));
  }
  PemModel m{model->alpha_p, model->beta_p, model->alpha_d, model->beta_d, cap, mns, mnbt};
  pem_batch_kernel<<<grid, kThreads>>>(n_sets, d_off, d_utok, d_rem, d_pre, m, d_scr, (int)max_items, d_out);
  RS_CUDA(cudaGetLastError());
  RS_CUDA(cudaMemcpy(values_out, d_out, n_sets * 8, cudaMemcpyDeviceToHost));
  cudaFree(d_off);
  cudaFree(d_utok);
  cudaFree(d_rem);
  cudaFree(d_pre);
  cudaFree(d_scr);
  cudaFree(d_out);
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

}  // extern "C"
