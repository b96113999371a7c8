/*
 * relsim_oracle.h -- CPU restatement of the reference scheduler (TEST INFRASTRUCTURE).
 *
 * This is the parity checker and the CPU baseline, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.  It restates relsim's engine loop
 * (pkg/src/relsim/engine.py:179-463), the DPU (priority.py:81-339), the ABA
 * (arranger.py:71-179), the trie prefix cache with its lazy LRU heap
 * (prefix_cache.py:41-176) and numpy's PCG64 Generator.choice(replace=False)
 * (numpy 2.3, the reference's only arithmetic dependency), single-threaded
 * and with the reference's per-iteration full scans, in plain C.
 *
 * Parity of this restatement is pinned by the tests/golden fixtures, generated
 * by running the real reference (tests/golden/make_golden.py).
 */
#ifndef RELSIM_ORACLE_H_
#define RELSIM_ORACLE_H_

#include <stdint.h>
#include "../include/relserve.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
  OR_REC_DPU = 1,       /* record every DPU record per iteration */
  OR_REC_WAITING = 2,   /* record the full waiting order per iteration */
  OR_REC_RNG = 4        /* record the DPU RNG state after each update */
};

typedef struct {
  int32_t rq;           /* trace-order relQuery index */
  int32_t reused;
  int32_t overridden;
  int32_t pad;
  double value;
} or_dpu_rec;

typedef struct {
  int32_t status;
  int32_t pad;
  int64_t iterations;
  double clock;
  int64_t cache_hit_tokens, cache_miss_tokens, kv_reserved;
  double dpu_wall_s, aba_wall_s, total_wall_s;
  double first_sight_wall_s;   /* wall time of the iteration that estimated the most relQueries */
  int64_t first_sight_iter;
  int64_t n_log;
  rs_iter_record* log;
  int64_t num_relqueries, num_requests;
  double *first_prefill_start, *last_prefill_end, *last_decode_end;  /* [R] NaN = None */
  int32_t* generated;          /* [N] */
  uint8_t* prefilled;          /* [N] */
  int64_t* completion_iter;    /* [N] */
  double* priority;            /* [N] */
  int64_t n_dpu;               /* OR_REC_DPU */
  int64_t* dpu_off;            /* [n_log+1] */
  or_dpu_rec* dpu;
  int64_t n_wait;              /* OR_REC_WAITING */
  int64_t* wait_off;           /* [n_log+1] */
  int32_t* wait;
  uint64_t* rng_trace;         /* OR_REC_RNG: [n_log][4] = state_hi, state_lo, has_uint32, uinteger */
  rs_pcg64_state rng;          /* final DPU RNG state */
  double* iter_wall;           /* [n_log] wall seconds per iteration */
  char message[256];
} or_result;

/*
 * Run the reference engine loop on one trace.  When path_off/path_node are
 * NULL the static trie is synthesised from chain_blocks (shared chain per
 * relQuery + private tail per row); otherwise row r's whole blocks map to
 * static trie nodes path_node[path_off[r] .. path_off[r+1]) whose parents
 * are node_parent[] (-1 = root).  Returns a heap-allocated result (free with
 * or_free) whose status is an RS_* code.
 */
or_result* or_run(const rs_trace_view* tr, const int64_t* path_off, const int32_t* path_node,
                  const int32_t* node_parent, int64_t n_nodes, const rs_config* cfg,
                  const rs_cost_model* world, const rs_cost_model* policy,
                  const rs_pcg64_state* rng, int32_t record_flags);

/* or_run with world-model noise: noise[k] is the standard normal the reference
   draws for its k-th executed batch (engine.py:310-313); needed when
   cfg->noise_sigma > 0. */
or_result* or_run_noise(const rs_trace_view* tr, const int64_t* path_off, const int32_t* path_node,
                        const int32_t* node_parent, int64_t n_nodes, const rs_config* cfg,
                        const rs_cost_model* world, const rs_cost_model* policy,
                        const rs_pcg64_state* rng, int32_t record_flags, const double* noise,
                        int64_t noise_len);

void or_free(or_result* r);

/* pem() over explicit items (priority.py:163-218). Returns RS_EINFEASIBLE on utok > cap. */
int or_pem(int64_t n, const int64_t* utok, const int32_t* remaining, const uint8_t* prefilled,
           int64_t cap, int64_t mns, int64_t mnbt, const rs_cost_model* m, double* out);

/* Generator.choice(n, k, replace=False) -> idx[k] (unshuffled order as numpy returns it). */
int or_choice(rs_pcg64_state* st, int64_t n, int64_t k, int64_t* idx);

/* Raw next64 / next32 (for RNG unit tests against numpy). */
uint64_t or_next64(rs_pcg64_state* st);
uint32_t or_next32(rs_pcg64_state* st);

#ifdef __cplusplus
}
#endif

#endif
