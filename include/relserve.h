/*
 * relserve.h -- C ABI of the B200-native RelServe scheduling hot path.
 *
 * The reference (`relsim`, pure Python) has no FFI; its "operator API" is the
 * Python call `relsim.engine.run(trace, policy, world_model, config,
 * policy_model, seed) -> RunResult` (pkg/src/relsim/engine.py:466-475) and the
 * `Engine(...)` class with the same constructor (engine.py:180-239).  This ABI
 * is what a binding for that call needs: plain pointers and sizes, no torch
 * types.  The Python package `paper_2601_11546_b200` binds it with ctypes
 * (see INTEGRATION.md for the binding a relsim maintainer would add).
 *
 * All entry points return an RS_* status code; rs_last_error() returns a
 * thread-local message for the last failure on the calling thread.
 */
#ifndef RELSERVE_H_
#define RELSERVE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (the Python shim re-raises the matching reference exception) */
enum {
  RS_OK = 0,
  RS_EINVAL = 1,          /* ValueError: bad policy/tau/constraints (engine.py:189-190, priority.py:36-40,250-251) */
  RS_EINFEASIBLE = 2,     /* InfeasibleRequestError: tok+output_limit > cap (engine.py:235-239) */
  RS_EABORT_LIMIT = 3,    /* SimulationAborted: iteration limit (engine.py:376-379) */
  RS_EABORT_IDLE = 4,     /* SimulationAborted: idle with live relQueries, no arrivals (engine.py:441-445) */
  RS_ECACHE_PINNED = 5,   /* RuntimeError: prefix cache cannot evict (prefix_cache.py:138) */
  RS_ECUDA = 6,           /* CUDA runtime failure */
  RS_ENOMEM = 7,
  RS_EUNSUPPORTED = 8,    /* input outside the device model (e.g. non-forest prefix structure) */
  RS_RUNNING = 100        /* trace not finished yet (status of a live trace) */
};

/* ---- policies (engine.py:45) */
enum {
  RS_POLICY_FCFS = 0,
  RS_POLICY_SP = 1,
  RS_POLICY_RELSERVE = 2,
  RS_POLICY_RELSERVE_PP = 3,
  RS_POLICY_RELSERVE_DP = 4
};

/* ---- decision enums (arranger.py:30-40) */
enum { RS_ACTION_PREFILL = 0, RS_ACTION_DECODE = 1, RS_ACTION_IDLE = 2 };
enum { RS_CASE_PREEMPT = 0, RS_CASE_INTERNAL = 1, RS_CASE_TRANSITIONAL = 2, RS_CASE_FORCED = 3 };

/* Iteration cost model alpha*x + beta (cost_model.py:23-58). */
typedef struct {
  double alpha_p, beta_p, alpha_d, beta_d;
} rs_cost_model;

/* EngineConfig (engine.py:141-158) + SchedulerConstraints (priority.py:30-40). */
typedef struct {
  int64_t cap;                    /* max resident tokens */
  int64_t max_num_seqs;           /* mns */
  int64_t max_num_batched_tokens; /* mnbt */
  int64_t sample_size;            /* DPU cache-miss sample size */
  double tau;                     /* starvation threshold (INFINITY disables) */
  double noise_sigma;             /* world-model noise (see rs_engine_set_noise) */
  int64_t block_size;             /* prefix-cache block (tokens) */
  int64_t capacity_blocks;        /* prefix-cache capacity (blocks) */
  int64_t iteration_limit;
  int32_t log_decisions;          /* record one rs_iter_record per iteration */
  int32_t policy;                 /* RS_POLICY_* */
  int32_t record_order;           /* parity mode: also snapshot every iteration's priority update
                                     (rs_engine_read_dpu) and waiting order (rs_engine_read_order);
                                     needs log_decisions; any number of relQueries */
  int32_t reserved;
} rs_config;

/* numpy PCG64 bit-generator state (`Generator.bit_generator.state`). */
typedef struct {
  uint64_t state_hi, state_lo;
  uint64_t inc_hi, inc_lo;
  uint32_t has_uint32, uinteger;
} rs_pcg64_state;

/*
 * One trace, column-wise, in trace order (the order of ArrivalTrace.entries).
 * Rows of relQuery i are row_off[i] .. row_off[i+1]-1 in req_id order.
 * chain_blocks[i] = number of leading whole blocks shared by every row of
 * relQuery i; all other blocks of a row are private to it (the prefix-cache
 * forest structure of generate_trace/load_trace traces).
 * static_prio may be NULL except for RS_POLICY_SP (static_relquery_prio,
 * priority.py:230-235, evaluated on the host because its mappings are
 * arbitrary callables in the reference).
 */
typedef struct {
  int64_t num_relqueries;
  int64_t num_requests;
  const int64_t* rel_id;        /* [R] */
  const double* arrival;        /* [R] */
  const int32_t* output_limit;  /* [R] */
  const int64_t* row_off;       /* [R+1] */
  const int32_t* tok;           /* [N] input tokens */
  const int32_t* out;           /* [N] actual_output_len (simulated EOS) */
  const int32_t* chain_blocks;  /* [R] */
  const double* static_prio;    /* [R] or NULL */
} rs_trace_view;

/*
 * One scheduler iteration (DecisionLogEntry, engine.py:64-74, plus what the
 * parity tests compare).  Optional floats are NaN when the reference has None.
 * relQuery indices are trace-order indices (map through rel_id[]).
 */
typedef struct {
  int64_t iteration;
  double clock;          /* clock when the decision was taken */
  double m_plus, m_minus;
  double delta_plus, delta_minus, delta_total;
  int64_t kv_reserved;   /* after execution */
  int32_t action;        /* RS_ACTION_* */
  int32_t kase;          /* RS_CASE_* */
  int32_t head;          /* waiting[0] relQuery index, -1 if none */
  int32_t n_waiting;     /* len(waiting) after the priority update */
  int32_t batch_rq;      /* prefill: relQuery index; else -1 */
  int32_t batch_first;   /* prefill: first req_id taken */
  int32_t batch_n;       /* prefill: rows taken; decode: batch size; idle: 0 */
  int32_t n_reestimated; /* relQueries whose priority was recomputed */
} rs_iter_record;

/* Per-trace progress/result summary (RunResult scalars, engine.py:77-102). */
typedef struct {
  int64_t iterations;
  double clock;                /* sim_duration when finished */
  int64_t cache_hit_tokens;
  int64_t cache_miss_tokens;
  int64_t kv_reserved;
  int64_t n_log;               /* decision records written so far */
  int64_t live_relqueries;
  int64_t admitted;
  int32_t status;              /* RS_RUNNING, RS_OK (finished) or an error code */
  int32_t error_detail;
  rs_pcg64_state rng;          /* DPU RNG state */
  /* device clock64() cycles per phase, summed over iterations: [0] admission,
     [1] priority update (DPU) remainder, [2] waiting order, [3] candidates +
     decision (ABA), [4] execution; finer marks [5..14] (see bench.py PHASES) */
  int64_t phase_cycles[23];
  /* bytes of request / FIFO / log state the iterations had to read or write in
     HBM (the relQuery table and running list live in shared memory) */
  int64_t alg_bytes;
  int64_t batches;             /* executed prefill/decode batches (= world-model noise draws consumed) */
} rs_trace_status;

typedef struct rs_engine rs_engine;

/* Last error message on this thread. */
const char* rs_last_error(void);

/* Library build/device info, e.g. "sm_100a". */
const char* rs_build_info(void);

/*
 * Create an engine over n_traces independent traces (one device scheduler
 * per trace) and upload their state to `device`.  Replaces the Engine
 * constructor (engine.py:180-239): validates the policy/config, rejects
 * infeasible requests, and seeds each trace's DPU RNG from rng[t] (numpy
 * `default_rng(SeedSequence([seed, 0xD9]))`, engine.py:224).
 * log_capacity = decision records kept per trace between rs_engine_read_log
 * calls (records beyond it are dropped; status.n_log still counts them).
 */
int rs_engine_create(const rs_trace_view* traces, int32_t n_traces, const rs_config* cfg,
                     const rs_cost_model* world, const rs_cost_model* policy_model,
                     const rs_pcg64_state* rng, int32_t device, int64_t log_capacity,
                     rs_engine** out);

/*
 * Advance every unfinished trace by up to max_iters scheduler iterations
 * (one pass of Engine.run's loop body, engine.py:375-448, each).  Enqueued
 * on `stream` (a cudaStream_t, NULL = legacy default); does not synchronize.
 */
int rs_engine_step(rs_engine* e, int64_t max_iters, void* stream);

/*
 * World-model noise (EngineConfig.noise_sigma > 0, engine.py:310-313): the
 * reference multiplies each executed batch's duration by 1 + sigma * z, z the
 * next standard normal of numpy default_rng(SeedSequence([seed, 0xE7])).  That
 * stream is independent of every scheduling decision, so the caller supplies
 * its first n values (z[k] for the k-th batch) for trace t (-1: every trace);
 * a launch that runs out stops early with RS_RUNNING and status.batches == n,
 * and the caller passes a longer prefix.  Required before stepping when
 * noise_sigma > 0.
 */
int rs_engine_set_noise(rs_engine* e, int32_t t, const double* z, int64_t n);

/* Synchronize `stream` and copy every trace's status to status[n_traces]. */
int rs_engine_status(rs_engine* e, void* stream, rs_trace_status* status);

/* Copy decision records [first, first+count) of trace t (must still be in the buffer). */
int rs_engine_read_log(rs_engine* e, int32_t t, int64_t first, int64_t count, rs_iter_record* out);

/*
 * Parity mode (cfg.record_order): the whole waiting queue after the priority
 * update of iterations [first, first+count) (engine.py:277-281: sorted by
 * (priority, arrival, rel_id)), as trace-order relQuery indices.  Row i of
 * out has `stride` = num_relqueries entries; its first record.n_waiting are
 * the queue, the rest -1.  The hot path never sorts: it only needs the head
 * and the length (a top-1 over a static order); the order is
 * rebuilt from the iteration's priority snapshot by the device radix sort
 * (rs_sort_pairs' kernels) when read.  count <= the log capacity; read the
 * rows of a launch before the next launch.
 */
int rs_engine_read_order(rs_engine* e, int32_t t, int64_t first, int64_t count, int32_t* out);

/*
 * Parity mode (cfg.record_order): the Dynamic Priority Updater's records of
 * iterations [first, first+count) (priority.py:287-315).  Row i of values /
 * flags has num_relqueries entries in trace order: the relQuery's priority
 * after the update (NaN if not admitted yet) and RS_SNAP_* bits; rng[i] is the
 * DPU generator state after the update.  Any pointer may be NULL.
 */
enum {
  RS_SNAP_ESTIMATED = 1,  /* recomputed this iteration (PriorityRecord.reused == False) */
  RS_SNAP_OVERRIDE = 2,   /* starvation override applied (priority.py:318-339) */
  RS_SNAP_LIVE = 4,       /* in live_relqueries: admitted and not retired */
  RS_SNAP_WAITING = 8     /* has pending rows: in the waiting queue */
};
int rs_engine_read_dpu(rs_engine* e, int32_t t, int64_t first, int64_t count, double* values, uint8_t* flags,
                       rs_pcg64_state* rng);
/* Timestamp ledgers per relQuery in trace order; NaN = None (engine.py:52-61). */
int rs_engine_read_ledgers(rs_engine* e, int32_t t, double* arrival, double* first_prefill_start,
                           double* last_prefill_end, double* last_decode_end);

/*
 * Per-request final state in trace order: generated tokens, prefilled flag,
 * completion iteration (-1 = not finished), and the last priority written.
 * Any pointer may be NULL.
 */
int rs_engine_read_requests(rs_engine* e, int32_t t, int32_t* generated, uint8_t* prefilled,
                            int64_t* completion_iter, double* priority);

/*
 * The running list between steps (Engine.running, engine.py:205, 326-329,
 * 358-359): the trace-order row index of every running request in execution
 * order.  Writes min(n_running, cap) rows and the full count to *n_running.
 */
int rs_engine_read_running(rs_engine* e, int32_t t, int32_t* rows, int32_t cap, int32_t* n_running);

/*
 * Every trace's results at once (multi-trace engines, e.g. a sweep of
 * independent traces): the ledgers' first_prefill_start / last_prefill_end /
 * last_decode_end (NaN = None) of all relQueries and the completion iteration
 * of all requests, traces concatenated in creation order, each in trace order
 * -- one page-locked batch of copies on `stream` and one synchronisation.
 * Any output pointer may be NULL.
 */
int rs_engine_read_results(rs_engine* e, void* stream, double* first_prefill_start, double* last_prefill_end,
                           double* last_decode_end, int32_t* completion_iter);
/*
 * Completion iteration per request (trace order, -1 = not finished) as int32:
 * the device column copied straight into `completion_iter` (page-locked
 * memory makes it one DMA).  The per-request output the reference's ledgers
 * are derived from (engine.py:358-362); the bulk result of a run.
 */
int rs_engine_read_completion(rs_engine* e, int32_t t, int32_t* completion_iter);

/* ---------------------------------------------------------------------------
 * Sharded pool (BASELINE config 5): one trace whose relQueries are
 * owned round-robin by admission rank across `shards` shards.  Each shard
 * keeps a full replica of the scheduler state and replays the same arranger
 * and state advance; it re-estimates only the partially prefilled relQueries
 * it owns and orders only its own waiting relQueries.  Once per scheduler
 * iteration the shards allgather one record each (local waiting head + the
 * priorities they computed) through peer memory inside the persistent kernel
 * (paper_2601_11546_b200/csrc/shard.cuh).  Decisions are bit-identical to the
 * unsharded engine.  Replaces nothing in the reference (which has no
 * parallel engine); it is the multi-GPU form of run() (engine.py:466-475).
 *
 *   rank == -1 : every shard in this engine, one CTA per shard on `device`
 *                (shards <= number of SMs); ready to step.
 *   rank >= 0  : this engine is shard `rank` only (one process per GPU);
 *                export rs_engine_mailbox() through rs_ipc_get_handle(),
 *                map the peers' with rs_ipc_open_handle(), call
 *                rs_engine_connect(), then step every shard with the same
 *                max_iters (each launch waits for its peers every iteration).
 * Status/log/ledger/request reads of any replica (t = 0) give the run's result.
 * ------------------------------------------------------------------------- */
int rs_engine_create_sharded(const rs_trace_view* trace, const rs_config* cfg, const rs_cost_model* world,
                             const rs_cost_model* policy_model, const rs_pcg64_state* rng, int32_t device,
                             int64_t log_capacity, int32_t shards, int32_t rank, rs_engine** out);

/* Device pointer and size of a one-shard engine's mailbox (to export). */
int rs_engine_mailbox(rs_engine* e, void** dptr, int64_t* bytes);

/* peer_mailboxes[shards]: every shard's mailbox as addressable from this
   engine's device (entry `rank` is ignored). */
int rs_engine_connect(rs_engine* e, void* const* peer_mailboxes);

/* CUDA IPC helpers (handle = 64 opaque bytes; cudaIpcMemHandle_t). */
int rs_ipc_get_handle(void* dptr, uint8_t* handle);
int rs_ipc_open_handle(const uint8_t* handle, int32_t device, void** dptr);
int rs_ipc_close(void* dptr);

/* Release all device memory of the engine. */
void rs_engine_destroy(rs_engine* e);

/* Device bytes held per trace (SoA + scratch), for reporting. */
int64_t rs_engine_device_bytes(const rs_engine* e);

/* SM clock of `device` in kHz (converts rs_trace_status.phase_cycles to seconds). */
int rs_device_clock_khz(int32_t device);

/* ---------------------------------------------------------------------------
 * relsim-trace-v1 ingestion (pkg/docs/trace-schema.md; workload.py:324-384):
 * the counts of a trace file as the columns rs_trace_view points at.  Host
 * code, no device needed.  Errors (bad schema, size != len(requests),
 * per-request prefix_len != the relQuery's) return RS_EINVAL with
 * rs_trace_v1_error() set.
 * ------------------------------------------------------------------------- */
typedef struct rs_trace_file rs_trace_file;
int rs_trace_v1_load(const char* path, rs_trace_file** out);
int rs_trace_v1_info(const rs_trace_file* f, int64_t* num_relqueries, int64_t* num_requests, double* rate,
                     int64_t* seed);
/* rel_id/arrival/output_limit/prefix_len [R], row_off [R+1], tok/out [N], trace (file) order */
int rs_trace_v1_columns(const rs_trace_file* f, int64_t* rel_id, double* arrival, int32_t* output_limit,
                        int32_t* prefix_len, int64_t* row_off, int32_t* tok, int32_t* out);
void rs_trace_v1_free(rs_trace_file* f);
const char* rs_trace_v1_error(void);

/* ---------------------------------------------------------------------------
 * Unit entry points (parity tests); same device code as the engine.
 * ------------------------------------------------------------------------- */

/*
 * pem() (priority.py:163-218) for n_sets remainders on the device.  Items of
 * set s are item_off[s] .. item_off[s+1]-1 in request order; utok is the
 * estimator's uncached-token count (0 if prefilled), remaining = decode
 * iterations left, prefilled in {0,1}.  Host buffers; synchronous.
 */
int rs_pem_batch(int64_t n_sets, const int64_t* item_off, const int64_t* utok,
                 const int32_t* remaining, const uint8_t* prefilled, int64_t cap,
                 int64_t max_num_seqs, int64_t max_num_batched_tokens,
                 const rs_cost_model* model, double* values_out, int32_t device);

/*
 * Unit entry point of the waiting order (engine.py:277-281 sort key
 * (priority, arrival, rel_id), of which the engine needs only the head and
 * len(waiting)): over n relQueries given in admission order -- sorted by
 * (arrival, rel_id), engine.py:211-213 -- the first minimum of `priority`
 * among those with waiting[i] != 0 (*head = -1 if none) and their count.  The
 * engine's own full-scan reduction on the device, over the order-preserving
 * key of each priority (any sign; NaN and -0.0 are EINVAL).
 * Replaces: the `waiting.sort(key=...)` + `waiting[0]` pair of Engine.run.
 */
int rs_waiting_argmin(const double* priority, const uint8_t* waiting, int64_t n, int32_t device, int64_t* head,
                      int64_t* count);

/*
 * The Adaptive Batch Arranger for given candidates (the engine's device code):
 * project_delta(prefill, output_limit_p, running, W, model) (arranger.py:115-143)
 * when both candidates are non-empty and m_plus <= m_minus, then decide_next
 * (arranger.py:146-179); fcfs/sp decide prefill-first (engine.py:387-395).
 * Running side: the n_run DISTINCT relQueries of the decode candidate (rel_id,
 * output_limit; any order -- sorted by rel_id on the device as engine.py:406-408
 * does), d_min_rel_id = rel_id of the first running request with the minimum
 * priority m_plus.  Prefill side: n_prefill requests with prefill_utok
 * uncached tokens of relQuery prefill_rel_id, priority m_minus.  An empty
 * candidate has n = 0 (its m is ignored).  n_waiting = len(waiting).  Writes
 * action, kase, m_plus, m_minus, delta_plus/minus/total (NaN = None),
 * n_waiting and batch_n of *out.  Host buffers; synchronous.
 */
int rs_arrange(int32_t n_run, const int64_t* run_rel_id, const int64_t* run_output_limit, int64_t d_min_rel_id,
               int32_t n_prefill, int64_t prefill_utok, int64_t prefill_rel_id, int64_t prefill_output_limit,
               double m_plus, double m_minus, int64_t n_waiting, int32_t policy, const rs_cost_model* model,
               int32_t device, rs_iter_record* out);

/*
 * numpy Generator.choice(n, k, replace=False) replay for a sequence of calls
 * (prefix_cache.py:157-158): call c draws k[c] of n[c] (k < n, Floyd path),
 * writing the k[c] indices at idx_out[off] (off = running sum of k).  The
 * final generator state is written back to *rng.  Host buffers; synchronous.
 */
int rs_choice_sequence(rs_pcg64_state* rng, int64_t n_calls, const int64_t* n, const int64_t* k,
                       int64_t* idx_out, int32_t device);

/*
 * North-star kernel 2 as a unit entry point: stable sort of n (key, value)
 * pairs by unsigned 64-bit key (equal keys keep their input order) with the
 * device LSD radix sort the engine uses for its static waiting order and
 * parity-mode waiting orders (csrc/radix_sort.cuh).  With keys =
 * order-preserving priority keys and values = admission ranks in rank order
 * this is `waiting.sort(key=sort_key)` (engine.py:175-176, 277-281).  Host
 * buffers; synchronous.
 */
int rs_sort_pairs(const uint64_t* keys, const int32_t* values, int64_t n, uint64_t* keys_out, int32_t* values_out,
                  int32_t device);

#ifdef __cplusplus
}
#endif

#endif /* RELSERVE_H_ */
