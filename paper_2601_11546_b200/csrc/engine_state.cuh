// engine_state.cuh -- device data layout of the scheduler.
//
// Per trace, in HBM (structure of arrays, indexed by admission rank -- the
// order relsim's DPU visits live relQueries, engine.py:211-213, 254, 279):
//   relQuery table  arrival, row offsets, output_limit, chain blocks, rel_id
//                   order, priority, prefilled prefix q, done/running counts,
//                   prefix-cache chain state (m, c0, ntails)
//   request rows    tok, out (EOS point), generated, completion iteration
//   prefix cache    FIFO of resident private tails (insertion order)
//   control block   clock, iteration, kv, queues, RNG, cache counters
// During a launch the control block and, when it fits, the whole relQuery
// table live in shared memory (RqView points at either copy).
#pragma once
#include <stdint.h>
#include <string.h>

#include "../../include/relserve.h"
#include "block.cuh"
#include "pcg64.cuh"
#include "pem.cuh"
#include "seg_pem.cuh"
#include "warp_pem.cuh"

namespace rsd {

struct ShardRec;  // shard.cuh

constexpr int kMaxRun = 1024;   // device limit on max_num_seqs
constexpr int kMaxAct = 1024;   // partially-prefilled live relQueries
constexpr int kMaxCC = 256;     // tail-less resident chains
constexpr int kWin = 768;       // FIFO window of the batched prefill eviction
constexpr int kEstBatch = 128;  // relQueries re-estimated per DPU batch
constexpr int kDrawBuf = 4096;  // numpy next32 draws staged per DPU batch
#ifndef RS_ITEM_BUF
#define RS_ITEM_BUF 1536  // keeps Shared below the 132 KB carve-out (a larger L1 for traces whose relQuery table is in HBM)
#endif
constexpr int kItemBuf = RS_ITEM_BUF;  // PEM items staged per segment-parallel batch
constexpr int kPhases = 24;
constexpr int kSmallEst = 32;   // DPU fast path: at most this many re-estimated relQueries
constexpr int kSmallMns = 256;  // ... and max_num_seqs at most this
constexpr int kMaxJobs = 64;    // ... and at most this many PEM segments
constexpr int kJobTerms = 32;   // fp64 terms per PEM segment kept in shared memory (the rest spill to HBM)
constexpr int kZScanRounds = 8;  // static-order scan: 32-entry rounds before the full reduction

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
  long long alg_bytes;  // HBM/L2 bytes the algorithm must move
  long long n_batch;    // executed batches = world-model noise draws consumed (engine.py:310-313)
  long long fifo_head, fifo_tail;
  int n_admitted, live;
  int n_run, n_act;
  int zptr, n_wait;  // static-order scan start (zl entries before it are prefilled); len(waiting)
  unsigned long long zh_key;  // cached static-order head (priority bits, rank) ...
  int zh_idx, zh_valid;       // ... valid until an admission or a prefill of that relQuery
  int status, error_detail;
  int cc_n, n_rrq;
  rs_pcg64_state rng;
  long long phase[kPhases];  // clock64 cycles per phase (+ scratch timestamp in the last slot)
  // running list (engine.py:205), in execution order, with the row state decode needs
  int run_row[kMaxRun];
  int run_rank[kMaxRun];
  int run_gen[kMaxRun];
  int run_out[kMaxRun];
  int run_kv[kMaxRun];   // tok + output_limit reserved by the row
  int act[kMaxAct];      // partially prefilled live relQueries, by rank
  int rrq[kMaxRun];      // relQueries with running rows (distinct)
  CcEnt cc[kMaxCC];
};
static_assert(sizeof(Ctl) % 16 == 0, "Ctl is copied as int4");

// relQuery table view (shared or global memory).
struct RqView {
  double* prio;
  double* arrival;
  unsigned long long* c0;
  int* off;  // [R+1]
  int* q;
  int* m;
  int* ntails;
  int* nrun;
  int* ndone;
  int* ol;
  int* chain;
  int* relrank;  // rank of the relQuery's rel_id among all rel_ids (tie order)
  int* scr_cnt;
  int* scr_last;
  int* zl;  // ranks sorted by (static priority bits, rank): the order of never-prefilled relQueries
};

// bytes of the relQuery table for R relQueries (16-byte aligned sections)
__host__ __device__ inline size_t rq_bytes(int R) {
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  return 3 * al(8 * (size_t)R) + al(4 * ((size_t)R + 1)) + 11 * al(4 * (size_t)R);
}

__host__ __device__ inline RqView rq_carve(void* base, int R) {
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  char* p = (char*)base;
  RqView v;
  v.prio = (double*)p;
  p += al(8 * (size_t)R);
  v.arrival = (double*)p;
  p += al(8 * (size_t)R);
  v.c0 = (unsigned long long*)p;
  p += al(8 * (size_t)R);
  v.off = (int*)p;
  p += al(4 * ((size_t)R + 1));
  int** ints[11] = {&v.q, &v.m, &v.ntails, &v.nrun, &v.ndone, &v.ol, &v.chain, &v.relrank, &v.scr_cnt, &v.scr_last,
                    &v.zl};
  for (int i = 0; i < 11; ++i) {
    *ints[i] = (int*)p;
    p += al(4 * (size_t)R);
  }
  return v;
}

// parity-mode snapshot flags per relQuery and iteration (rs_engine_read_dpu)
constexpr unsigned char kSnapEstimated = 1;  // priority recomputed this iteration (not reused, priority.py:296-303)
constexpr unsigned char kSnapOverride = 2;   // starvation override applied (priority.py:318-339)
constexpr unsigned char kSnapLive = 4;       // in live_relqueries (admitted, not retired; engine.py:254, 362)
constexpr unsigned char kSnapWaiting = 8;    // has pending (unprefilled) rows: in the waiting queue (engine.py:280)

struct TraceDev {
  int R, N, max_size, seg_ok;  // seg_ok: mns * max(tok) <= cap (PEM segments close by count only)
  int rq_in_smem, pad0;
  void* rq_global;             // relQuery table (rq_carve layout)
  const int* tok;              // [N] rank-ordered rows
  const int* out;
  int* gen;
  int* comp;
  double* fps;
  double* lpe;
  double* lde;
  FifoEnt* fifo;
  long long fifo_cap;
  const JumpEntry* jump;  // PCG64 jump-ahead table of this trace's DPU generator: [kJumpBits] powers of two, then 32 consecutive steps
  double* term_spill;     // [kMaxJobs * (kSmallMns + 1)] PEM terms beyond kJobTerms per segment
  const double* fsprio;   // [R] first-sight priority (static: no prefilled row, cold chain, ratio 1.0)
  const long long* fs_doff;  // [R+1] prefix of first-sight draw counts (2S-1 per relQuery larger than S)
  const int* ne_pref;        // [R+1] prefix count of relQueries with rows (waiting entries at admission)
  int fast;                  // engine_kernel<true> applies (see host)
  int nzl;                   // entries of rq.zl (this shard's relQueries)
  int shard_world, shard_rank;  // sharded pool: relQuery a is owned by shard a % world (1, 0: unsharded)
  int pad1;
  ShardRec* self_mbox;       // this shard's mailbox ShardRec[world][2] (shard.cuh)
  ShardRec* const* peers;    // [world] every shard's mailbox, as addressable from this device
  const double* noise;       // world-model noise: standard normals of the SeedSequence([seed, 0xE7]) stream
  long long noise_n;         // ... available (rs_engine_set_noise)
  rs_iter_record* log;
  long long log_cap;
  // parity mode (cfg.record_order), per logged iteration (row = n_log & (log_cap - 1)):
  double* snap_prio;            // [log_cap][R] every admitted relQuery's priority after the update (NaN: not admitted)
  unsigned char* snap_flag;     // [log_cap][R] kSnap* bits
  rs_pcg64_state* snap_rng;     // [log_cap] the DPU generator after the update
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
  int zorder;  // waiting head from the static order (no starvation override possible)
  long long max_iters;
  unsigned long long mns_magic;  // floor(2^32 / max_num_seqs) + 1: x / mns == (x * magic) >> 32 for x < 2^32 / mns
  unsigned dper_magic;           // floor(2^16 / (2*sample_size - 1)) + 1: the same for draw positions < 2^16 / dper
  int pad3;
};

struct Shared {
  Ctl c;
  RqView rq;
  ArgminSmem am;
  ScanSmem scan;
  Scan32Smem s32;
  RedSmem red;
  SegShared segsh;
  JumpEntry jt[kJumpBits];
  JumpEntry jstep[32];  // (A^k, C_k) for k = 1..32 steps
  int go, action;
  int go_exec;  // the pipelined iteration's execution result (group M -> everyone after the join)
  int go_admit;  // phase A's continue flag (separate from `go`: no barrier closes an iteration)
  int new_lo, new_hi;
  int head, W, taken, J;
  int pf_head;  // the previous iteration's head (candidate-row prefetch), set at the iteration end
  long long utok_sum;
  double m_plus, m_minus;
  int dmin_slot, n_est;
  unsigned long long sh_key[32];  // sharded pool: the shards' waiting heads of this iteration
  int sh_idx[32];
  int n_dist, act_dirty, rrq_dirty;
  double dterm[kMaxRun];  // projection terms of the distinct running relQueries, rel_id order
  int max_ol;             // ... and their largest output limit (reset after each use)
  int cand_tok[kMaxRun];  // staged candidate prefill rows (tok, out)
  int cand_out[kMaxRun];
  int cand_u[kMaxRun];     // inclusive utok prefix of the candidate rows
  int first_bad, cand_mh;
  // a candidate scanned after a decode (engine.cu), in its own 32-byte block: phase D
  // reads it while thread 0 writes the fields around (no vector load may straddle them)
  struct alignas(32) PreCand {
    int valid, head, J, mh, first_bad, pad[3];
  } pc;
  // DPU batch
  int est_rank[kEstBatch], est_off[kEstBatch], est_q[kEstBatch], est_nunp[kEstBatch];
  int est_ol[kEstBatch], est_m[kEstBatch], est_doff[kEstBatch + 1];
  int est_io[kEstBatch + 1], est_jo[kEstBatch + 1];  // PEM item / job offsets
  int est_drawer[kSmallEst];                          // k-th relQuery with choice() draws (fast path)
  double est_ratio[kEstBatch];
  PrefixSummary est_ps[kEstBatch];
  int rng_reject;
  uint32_t floyd_idx[kMaxSample];  // thread 0's sequential numpy choice() replays (cold paths)
  unsigned long long rej_pos;  // first-sight replay: first stream position with a Lemire rejection
  int new_lo_rs;               // ... and the arrival its parallel replay restarts at
  // pipelined priority update (common configuration): group D computes the next
  // iteration's update of the partially prefilled relQueries during this
  // iteration's state advance (dpu.cuh dpu_spec); committed after the join
  int spec_ok;    // this iteration's update of c.act is already done (committed)
  int spec_valid; // group D's verdict on its result (fits the fast path, no Lemire rejection)
  int spec_action; // the action the update assumed (certain, or the speculated prefill)
  int spec_n;     // entries of the speculative list
  int spec_rank[kSmallEst];
  int spec_m[kSmallEst];     // chain length its ratio assumed (checked against the advance's)
  int spec_nunp[kSmallEst];  // unprefilled rows after the advance
  int spec_base[kSmallEst];  // first unprefilled row
  int spec_ol[kSmallEst];
  int spec_L[kSmallEst];     // running rows after the advance: count, sum and max of remaining
  int spec_rsum[kSmallEst];
  int spec_rmax[kSmallEst];
  double spec_val[kSmallEst];
  rs_pcg64_state spec_rng;
  long long spec_alg;
  int spec_draws;  // next32 values the speculative update draws
  int spec_jobs;   // its PEM segments
  // batched prefill eviction
  int fp_bad, fp_popped, fp_par, fp_cut;
  long long fp_rem;
  unsigned long long fp_c0_last;
  union {
    unsigned int draws[kDrawBuf];
    struct {
      long long U[kItemBuf];
      double terms[2 * kItemBuf + kEstBatch];
      int UNP[kItemBuf];
      int REM[kItemBuf];
      int jcnt[kItemBuf + kEstBatch];
    } seg;
    struct {  // side by side: the pipelined iteration runs the DPU fast path and the prefill advance at once
      struct {
        unsigned int draws[kSmallEst * 31];
        alignas(16) double terms[kMaxJobs * kJobTerms];  // read two at a time by the ordered sums
        int nterm[kMaxJobs];
        int U[kWarps][kSmallMns];  // per-warp utok prefix of the segment it evaluates
      } small;
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
  // kPart (engine_kernel<true, true, true>) only; last, so the other fields keep their offsets
  int spec_part;  // the speculative list is the first kSmallEst entries of a longer one
  int spec_e0;    // after a partial commit: the first entry phase B estimates in place (else -1)
  // relQuery table follows (dynamic shared memory) when rq_in_smem
};

// Order-preserving 64-bit key of a priority: unsigned comparison of okey(x)
// equals numeric comparison of x for every non-NaN double (negative values:
// all bits flipped; others: sign bit set).  The engine's own priorities are
// non-negative, but sp's user-supplied static priorities may be negative
// (priority.py:221-235).  -0.0 never reaches the device (the host
// canonicalises static priorities; PEM sums start at +0.0).  Host twin:
// engine.cu order_key().
__host__ __device__ __forceinline__ unsigned long long okey(double x) {
#ifdef __CUDA_ARCH__
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
#else
  unsigned long long b;
  memcpy(&b, &x, 8);
#endif
  return b ^ ((unsigned long long)((long long)b >> 63) | 0x8000000000000000ULL);
}

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7FF8000000000000LL); }

// thread 0 accumulates the cycles since the previous mark into phase k.
// RS_PHASE_TIMERS: 0 off, 1 the five coarse phases (0-4: admission, DPU,
// waiting order, candidates + decision, execution), 2 also the fine marks.
#ifndef RS_PHASE_TIMERS
#define RS_PHASE_TIMERS 1
#endif
__device__ __forceinline__ void phase_mark(Ctl& c, int k) {
#if RS_PHASE_TIMERS >= 2
  // the clock read waits for a shared-memory load, which cannot complete before
  // a preceding barrier does (a bare read may retire under BAR.SYNC.DEFER_BLOCKING
  // and charge the barrier wait to the next phase)
  if (threadIdx.x == 0) {
    const long long prev = *(volatile long long*)&c.phase[kPhases - 1];
    long long now = prev;
    if (prev != 0x7FFFFFFFFFFFFFFFLL) now = clock64();
    c.phase[k] += now - prev;
    c.phase[kPhases - 1] = now;
  }
#elif RS_PHASE_TIMERS
  if (k < 5) {  // coarse phases only (each may absorb the tail of the preceding barrier wait)
    if (threadIdx.x == 0) {
      const long long now = clock64();
      c.phase[k] += now - c.phase[kPhases - 1];
      c.phase[kPhases - 1] = now;
    }
  }
#else
  (void)c;
  (void)k;
#endif
}

// Group D's own marks (slots 19-21, scratch stamp in slot 22) when built with
// -DRS_DPHASE=1: the pipelined priority update's list + summaries, metadata +
// RNG + ratios, PEM + ordered sums.
#ifndef RS_DPHASE
#define RS_DPHASE 0
#endif
// -DRS_DPHASE=2 (with RS_PHASE_TIMERS=1): also fine marks in slots 5-14.
__device__ __forceinline__ void dphase_mark(Ctl& c, int k) {
#if RS_DPHASE
  if (RS_DPHASE < 2 && k >= 5 && k < 19) return;
  if (threadIdx.x == kMWarps * 32) {
    const long long now = clock64();
    if (k >= 0) c.phase[k] += now - c.phase[22];
    c.phase[22] = now;
  }
#else
  (void)c;
  (void)k;
#endif
}

}  // namespace rsd
