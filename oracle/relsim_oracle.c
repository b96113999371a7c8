/*
 * relsim_oracle.c -- CPU restatement of the reference scheduler.
 *
 * TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).  See
 * relsim_oracle.h.  Every function cites the reference code it restates;
 * the control flow deliberately keeps the reference's per-iteration full
 * scans (priority.py:266, :307, :309-312; engine.py:280-281) so that timing
 * this file is timing the reference's algorithm, not a smarter one.
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off: CPython rounds every
 * * and + separately, so no FMA contraction is allowed).
 */
#include "relsim_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------ */
/* numpy PCG64 (pcg_setseq_128_xsl_rr_64) + Generator.choice(replace=False)  */
/* ------------------------------------------------------------------------ */

static const u128 PCG_MULT = (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;

static inline uint64_t rotr64(uint64_t v, unsigned r) { return (v >> r) | (v << ((64u - r) & 63u)); }

uint64_t or_next64(rs_pcg64_state* st) {
  u128 s = (((u128)st->state_hi) << 64) | st->state_lo;
  u128 inc = (((u128)st->inc_hi) << 64) | st->inc_lo;
  s = s * PCG_MULT + inc; /* step first, then output the new state */
  st->state_hi = (uint64_t)(s >> 64);
  st->state_lo = (uint64_t)s;
  return rotr64(st->state_hi ^ st->state_lo, (unsigned)(st->state_hi >> 58));
}

uint32_t or_next32(rs_pcg64_state* st) {
  if (st->has_uint32) {
    st->has_uint32 = 0;
    return st->uinteger;
  }
  uint64_t v = or_next64(st);
  st->has_uint32 = 1;
  st->uinteger = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

/* random_bounded_uint64(off=0, rng, use_masked=0) for rng < 2^32: Lemire on 32-bit draws. */
static uint64_t bounded32(rs_pcg64_state* st, uint64_t rng) {
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFULL) return or_next32(st);
  const uint32_t excl = (uint32_t)rng + 1u;
  uint64_t m = (uint64_t)or_next32(st) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t thr = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % excl;
    while (left < thr) {
      m = (uint64_t)or_next32(st) * excl;
      left = (uint32_t)m;
    }
  }
  return m >> 32;
}

/* Generator.choice(n, k, replace=False, shuffle=True): Floyd's algorithm, then
 * a Fisher-Yates pass over the k results (numpy _generator.pyx).  Only the
 * Floyd branch (not n > 10000 and k > n // 50) is restated. */
int or_choice(rs_pcg64_state* st, int64_t n, int64_t k, int64_t* idx) {
  if (k < 0 || k > n) return RS_EINVAL;
  if (n > 0xFFFFFFFFLL) return RS_EUNSUPPORTED;
  if (n > 10000 && k > n / 50) return RS_EUNSUPPORTED;
  for (int64_t j = n - k; j < n; ++j) {
    int64_t v = (int64_t)bounded32(st, (uint64_t)j);
    int64_t pos = j - (n - k);
    int found = 0;
    for (int64_t q = 0; q < pos; ++q)
      if (idx[q] == v) { found = 1; break; }
    idx[pos] = found ? j : v;
  }
  for (int64_t i = k - 1; i >= 1; --i) {
    int64_t jj = (int64_t)bounded32(st, (uint64_t)i);
    int64_t t = idx[jj];
    idx[jj] = idx[i];
    idx[i] = t;
  }
  return RS_OK;
}

/* ------------------------------------------------------------------------ */
/* pem(): analytic Alg. 1 cost (priority.py:163-218)                        */
/* ------------------------------------------------------------------------ */

int or_pem(int64_t n, const int64_t* utok, const int32_t* remaining, const uint8_t* prefilled,
           int64_t cap, int64_t mns, int64_t mnbt, const rs_cost_model* m, double* out) {
  double total = 0.0;
  int64_t p_utok = 0, d_count = 0, d_sum = 0, d_max = 0, accum = 0;
  int p_nonempty = 0;
#define OR_FLUSH_SEGMENT()                                                   \
  do {                                                                       \
    if (p_nonempty) total += m->alpha_p * (double)p_utok + m->beta_p;        \
    if (d_count) total += m->alpha_d * (double)d_sum + m->beta_d * (double)d_max; \
    p_utok = 0; p_nonempty = 0; d_count = 0; d_sum = 0; d_max = 0; accum = 0; \
  } while (0)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t u = utok[i];
    if (u > cap) return RS_EINFEASIBLE;
    if (u + accum > cap || d_count + 1 > mns) OR_FLUSH_SEGMENT();
    if (u > 0 && u + p_utok > mnbt) {
      if (p_nonempty) total += m->alpha_p * (double)p_utok + m->beta_p;
      p_utok = 0;
      p_nonempty = 0;
    }
    if (!prefilled[i]) {
      p_nonempty = 1;
      p_utok += u;
    }
    if (remaining[i] > 0) {
      d_count += 1;
      d_sum += remaining[i];
      if (remaining[i] > d_max) d_max = remaining[i];
    }
    accum += u;
  }
  OR_FLUSH_SEGMENT();
#undef OR_FLUSH_SEGMENT
  *out = total;
  return RS_OK;
}

/* ------------------------------------------------------------------------ */
/* Trie prefix cache with lazy LRU heap (prefix_cache.py:41-138)             */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint64_t access;
  int32_t node;
} hent;

typedef struct {
  int64_t B, C, count;
  uint64_t clock;
  int64_t n_nodes;
  const int32_t* parent;
  uint8_t* resident;
  uint64_t* last_access;
  int32_t* nres_child;
  uint32_t* pin;
  uint32_t pin_epoch;
  hent* heap;
  int64_t hn, hcap;
  hent* skipped;
  int64_t scap;
  int64_t hit_total, miss_total;
} cache_t;

static int heap_push(cache_t* c, hent e) {
  if (c->hn == c->hcap) {
    int64_t nc = c->hcap ? c->hcap * 2 : 1024;
    hent* h = (hent*)realloc(c->heap, (size_t)nc * sizeof(hent));
    if (!h) return -1;
    c->heap = h;
    c->hcap = nc;
  }
  int64_t i = c->hn++;
  while (i > 0) {
    int64_t p = (i - 1) >> 1;
    if (c->heap[p].access <= e.access) break;
    c->heap[i] = c->heap[p];
    i = p;
  }
  c->heap[i] = e;
  return 0;
}

static hent heap_pop(cache_t* c) {
  hent top = c->heap[0];
  hent last = c->heap[--c->hn];
  int64_t i = 0, n = c->hn;
  for (;;) {
    int64_t l = 2 * i + 1;
    if (l >= n) break;
    int64_t s = (l + 1 < n && c->heap[l + 1].access < c->heap[l].access) ? l + 1 : l;
    if (c->heap[s].access >= last.access) break;
    c->heap[i] = c->heap[s];
    i = s;
  }
  if (n > 0) c->heap[i] = last;
  return top;
}

static int touch(cache_t* c, int32_t node) { /* prefix_cache.py:65-68 */
  c->clock += 1;
  c->last_access[node] = c->clock;
  hent e = {c->clock, node};
  return heap_push(c, e);
}

/* match_uncached (prefix_cache.py:70-93): walk leading resident blocks. */
static int64_t cache_match(cache_t* c, const int32_t* path, int64_t nb, int64_t tok, int refresh,
                           int record) {
  int64_t matched = 0;
  for (int64_t j = 0; j < nb; ++j) {
    int32_t node = path[j];
    if (!c->resident[node]) break;
    matched += 1;
    if (refresh) touch(c, node);
  }
  int64_t hit = matched * c->B;
  if (record) {
    c->hit_total += hit;
    c->miss_total += tok - hit;
  }
  return tok - hit;
}

/* _evict_one (prefix_cache.py:122-138). */
static int cache_evict_one(cache_t* c) {
  int64_t ns = 0;
  while (c->hn > 0) {
    hent e = heap_pop(c);
    int32_t node = e.node;
    if (c->last_access[node] != e.access || !c->resident[node]) continue; /* stale / evicted */
    if (c->nres_child[node] > 0 || c->pin[node] == c->pin_epoch) {
      if (ns == c->scap) {
        int64_t nc = c->scap ? c->scap * 2 : 256;
        hent* s = (hent*)realloc(c->skipped, (size_t)nc * sizeof(hent));
        if (!s) return RS_ENOMEM;
        c->skipped = s;
        c->scap = nc;
      }
      c->skipped[ns++] = e;
      continue;
    }
    c->resident[node] = 0;
    c->count -= 1;
    if (c->parent[node] >= 0) c->nres_child[c->parent[node]] -= 1;
    for (int64_t i = 0; i < ns; ++i) heap_push(c, c->skipped[i]);
    return RS_OK;
  }
  return RS_ECACHE_PINNED;
}

/* insert (prefix_cache.py:95-120). */
static int cache_insert(cache_t* c, const int32_t* path, int64_t nb) {
  if (nb > c->C) nb = c->C; /* truncated insert */
  c->pin_epoch += 1;
  for (int64_t j = 0; j < nb; ++j) {
    int32_t node = path[j];
    if (!c->resident[node]) {
      c->resident[node] = 1;
      c->count += 1;
      if (c->parent[node] >= 0) c->nres_child[c->parent[node]] += 1;
    }
    c->pin[node] = c->pin_epoch;
    touch(c, node);
  }
  while (c->count > c->C) {
    int rc = cache_evict_one(c);
    if (rc) return rc;
  }
  return RS_OK;
}

/* ------------------------------------------------------------------------ */
/* Engine (engine.py:179-463)                                               */
/* ------------------------------------------------------------------------ */

typedef struct {
  int32_t rq;
  int64_t pend;  /* pending = rows [pend, size) of rq: the taken batch is always a leading run */
} wentry;

typedef struct {
  const rs_trace_view* tr;
  const rs_config* cfg;
  const rs_cost_model* world;
  const rs_cost_model* pol;
  int64_t R, N;
  const int64_t* off;
  /* static trie paths */
  const int64_t* path_off;
  const int32_t* path_node;
  /* row state */
  uint8_t* prefilled;
  int32_t* gen;
  double* prio;
  int64_t* completion;
  /* relQuery state */
  uint8_t* live;
  uint8_t* seen_last;     /* in the previous update's records (priority.py:264) */
  double* rec_value;
  double* new_value;
  uint8_t* new_reused;
  uint8_t* new_override;
  int32_t* order;         /* admission order */
  int64_t next_arrival;
  int64_t n_live;
  wentry* waiting;
  int64_t n_waiting;
  int32_t* running;
  int64_t n_running;
  int64_t kv_reserved;
  double clock;
  int64_t iteration;
  rs_pcg64_state rng;
  cache_t cache;
  /* scratch */
  int64_t* s_utok;
  int32_t* s_rem;
  uint8_t* s_pre;
  int32_t* s_rows;
  int64_t* s_idx;
  int32_t* s_rels;
  /* sort context */
  const double* sort_arrival;
  const int64_t* sort_relid;
} eng_t;

static eng_t* g_sort_eng; /* qsort has no context pointer; the oracle is single-threaded */

static int cmp_arrival(const void* a, const void* b) {
  int32_t i = *(const int32_t*)a, j = *(const int32_t*)b;
  const rs_trace_view* t = g_sort_eng->tr;
  if (t->arrival[i] < t->arrival[j]) return -1;
  if (t->arrival[i] > t->arrival[j]) return 1;
  return (t->rel_id[i] > t->rel_id[j]) - (t->rel_id[i] < t->rel_id[j]);
}

/* _WaitingEntry.sort_key (engine.py:171-176): (pending[0].priority, arrival, rel_id). */
static int cmp_waiting(const void* a, const void* b) {
  const wentry* x = (const wentry*)a;
  const wentry* y = (const wentry*)b;
  const eng_t* e = g_sort_eng;
  double px = e->prio[e->off[x->rq] + x->pend], py = e->prio[e->off[y->rq] + y->pend];
  if (px < py) return -1;
  if (px > py) return 1;
  double ax = e->tr->arrival[x->rq], ay = e->tr->arrival[y->rq];
  if (ax < ay) return -1;
  if (ax > ay) return 1;
  int64_t rx = e->tr->rel_id[x->rq], ry = e->tr->rel_id[y->rq];
  return (rx > ry) - (rx < ry);
}

static inline int row_done(const eng_t* e, int64_t r) { return e->gen[r] >= e->tr->out[r]; }
static inline int64_t row_nb(const eng_t* e, int64_t r) { return e->path_off[r + 1] - e->path_off[r]; }
static inline const int32_t* row_path(const eng_t* e, int64_t r) { return e->path_node + e->path_off[r]; }
static inline int32_t row_rq_ol(const eng_t* e, int32_t rq) { return e->tr->output_limit[rq]; }

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* DynamicPriorityUpdater.estimate (priority.py:268-285). */
static int dpu_estimate(eng_t* e, int32_t rq, double* out) {
  const int64_t lo = e->off[rq], hi = e->off[rq + 1];
  int64_t n_live = 0, n_unp = 0;
  for (int64_t r = lo; r < hi; ++r)
    if (!row_done(e, r)) {
      n_live++;
      if (!e->prefilled[r]) e->s_rows[n_unp++] = (int32_t)r;
    }
  if (!n_live) {
    *out = 0.0;
    return RS_OK;
  }
  double ratio = 0.0;
  if (n_unp) {
    /* sample_cache_miss_ratio (prefix_cache.py:141-169) */
    int64_t k = e->cfg->sample_size < n_unp ? e->cfg->sample_size : n_unp;
    if (k < n_unp) {
      int rc = or_choice(&e->rng, n_unp, k, e->s_idx);
      if (rc) return rc;
    } else {
      for (int64_t i = 0; i < n_unp; ++i) e->s_idx[i] = i;
    }
    int64_t usum = 0, tsum = 0;
    for (int64_t i = 0; i < k; ++i) {
      int64_t r = e->s_rows[e->s_idx[i]];
      usum += cache_match(&e->cache, row_path(e, r), row_nb(e, r), e->tr->tok[r], 0, 0);
      tsum += e->tr->tok[r];
    }
    ratio = (double)usum / (double)tsum;
  }
  /* remainder_items (priority.py:81-98) with utok_approx (prefix_cache.py:172-176) */
  int64_t n = 0;
  const int32_t ol = row_rq_ol(e, rq);
  for (int64_t r = lo; r < hi; ++r) {
    int32_t rem = ol - e->gen[r];
    if (row_done(e, r) || (e->prefilled[r] && rem <= 0)) continue;
    int64_t u = 0;
    if (!e->prefilled[r]) {
      int64_t tok = e->tr->tok[r];
      int64_t a = (int64_t)floor((double)tok * ratio + 0.5);
      u = tok < a ? tok : a;
    }
    e->s_utok[n] = u;
    e->s_rem[n] = rem;
    e->s_pre[n] = e->prefilled[r];
    n++;
  }
  return or_pem(n, e->s_utok, e->s_rem, e->s_pre, e->cfg->cap, e->cfg->max_num_seqs,
                e->cfg->max_num_batched_tokens, e->pol, out);
}

/* DynamicPriorityUpdater.update (priority.py:287-315) + starvation (318-339). */
static int dpu_update(eng_t* e, int64_t* n_est, int32_t rec_flags, or_result* res) {
  const int64_t admitted = e->next_arrival;
  *n_est = 0;
  for (int64_t a = 0; a < admitted; ++a) {
    int32_t rq = e->order[a];
    if (!e->live[rq]) continue;
    int reuse = 0;
    if (e->seen_last[rq]) { /* _can_reuse (priority.py:261-266) */
      reuse = 1;
      for (int64_t r = e->off[rq]; r < e->off[rq + 1]; ++r)
        if (e->prefilled[r] || row_done(e, r)) {
          reuse = 0;
          break;
        }
    }
    e->new_override[rq] = 0;
    if (reuse) {
      e->new_value[rq] = e->rec_value[rq];
      e->new_reused[rq] = 1;
    } else {
      int rc = dpu_estimate(e, rq, &e->new_value[rq]);
      if (rc) return rc;
      e->new_reused[rq] = 0;
      (*n_est)++;
    }
  }
  if (isfinite(e->cfg->tau)) {
    for (int64_t a = 0; a < admitted; ++a) {
      int32_t rq = e->order[a];
      if (!e->live[rq]) continue;
      int any_pre = 0;
      for (int64_t r = e->off[rq]; r < e->off[rq + 1]; ++r)
        if (e->prefilled[r]) {
          any_pre = 1;
          break;
        }
      if (any_pre) continue;
      double unit_waiting = (e->clock - e->tr->arrival[rq]) / (double)(e->off[rq + 1] - e->off[rq]);
      if (unit_waiting > e->cfg->tau) {
        e->new_value[rq] = 0.0;
        e->new_override[rq] = 1;
      }
    }
  }
  for (int64_t a = 0; a < admitted; ++a) {
    int32_t rq = e->order[a];
    if (!e->live[rq]) continue;
    for (int64_t r = e->off[rq]; r < e->off[rq + 1]; ++r) e->prio[r] = e->new_value[rq];
  }
  for (int64_t a = 0; a < admitted; ++a) {
    int32_t rq = e->order[a];
    e->seen_last[rq] = e->live[rq];
    e->rec_value[rq] = e->new_value[rq];
  }
  if (rec_flags & OR_REC_DPU) {
    for (int64_t a = 0; a < admitted; ++a) {
      int32_t rq = e->order[a];
      if (!e->live[rq]) continue;
      if (res->n_dpu % 4096 == 0) {
        or_dpu_rec* d = (or_dpu_rec*)realloc(res->dpu, (size_t)(res->n_dpu + 4096) * sizeof(or_dpu_rec));
        if (!d) return RS_ENOMEM;
        res->dpu = d;
      }
      or_dpu_rec* d = &res->dpu[res->n_dpu++];
      d->rq = rq;
      d->reused = e->new_reused[rq];
      d->overridden = e->new_override[rq];
      d->pad = 0;
      d->value = e->new_value[rq];
    }
  }
  return RS_OK;
}

static void set_err(or_result* r, int code, const char* msg) {
  r->status = code;
  snprintf(r->message, sizeof r->message, "%s", msg);
}

static int grow(void** p, int64_t* cap, int64_t need, size_t elem) {
  if (need <= *cap) return 0;
  int64_t nc = *cap ? *cap : 1024;
  while (nc < need) nc *= 2;
  void* q = realloc(*p, (size_t)nc * elem);
  if (!q) return -1;
  *p = q;
  *cap = nc;
  return 0;
}

or_result* or_run(const rs_trace_view* tr, const int64_t* path_off_in, const int32_t* path_node_in,
                  const int32_t* node_parent_in, int64_t n_nodes_in, const rs_config* cfg,
                  const rs_cost_model* world, const rs_cost_model* policy,
                  const rs_pcg64_state* rng, int32_t rec_flags) {
  return or_run_noise(tr, path_off_in, path_node_in, node_parent_in, n_nodes_in, cfg, world, policy, rng,
                      rec_flags, NULL, 0);
}

/* _world_duration (engine.py:310-313): base * (1 + sigma * z) clamped at 0.0,
   z = the k-th standard normal of the engine's SeedSequence([seed, 0xE7])
   stream for the k-th executed batch (numpy's draws, passed in). */
static double world_duration(const rs_config* cfg, const double* noise, int64_t noise_len, int64_t* k,
                             double base, int* ok) {
  if (cfg->noise_sigma > 0) {
    if (*k >= noise_len) {
      *ok = 0;
      return base;
    }
    const double v = base * (1.0 + cfg->noise_sigma * noise[(*k)++]);
    base = v > 0.0 ? v : 0.0; /* max(0.0, v) */
  }
  return base;
}

or_result* or_run_noise(const rs_trace_view* tr, const int64_t* path_off_in, const int32_t* path_node_in,
                        const int32_t* node_parent_in, int64_t n_nodes_in, const rs_config* cfg,
                        const rs_cost_model* world, const rs_cost_model* policy,
                        const rs_pcg64_state* rng, int32_t rec_flags, const double* noise, int64_t noise_len) {
  or_result* res = (or_result*)calloc(1, sizeof(or_result));
  if (!res) return NULL;
  const int64_t R = tr->num_relqueries, N = tr->num_requests;
  res->num_relqueries = R;
  res->num_requests = N;
  res->first_prefill_start = (double*)malloc(sizeof(double) * (size_t)(R ? R : 1));
  res->last_prefill_end = (double*)malloc(sizeof(double) * (size_t)(R ? R : 1));
  res->last_decode_end = (double*)malloc(sizeof(double) * (size_t)(R ? R : 1));
  res->generated = (int32_t*)calloc((size_t)(N ? N : 1), sizeof(int32_t));
  res->prefilled = (uint8_t*)calloc((size_t)(N ? N : 1), 1);
  res->completion_iter = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N ? N : 1));
  res->priority = (double*)calloc((size_t)(N ? N : 1), sizeof(double));
  for (int64_t i = 0; i < R; ++i)
    res->first_prefill_start[i] = res->last_prefill_end[i] = res->last_decode_end[i] = NAN;
  for (int64_t i = 0; i < N; ++i) res->completion_iter[i] = -1;

  const int pol = cfg->policy;
  if (pol < RS_POLICY_FCFS || pol > RS_POLICY_RELSERVE_DP) {
    set_err(res, RS_EINVAL, "unknown policy");
    return res;
  }
  if (cfg->cap <= 0 || cfg->max_num_seqs <= 0 || cfg->max_num_batched_tokens <= 0) {
    set_err(res, RS_EINVAL, "constraints must be positive");
    return res;
  }
  if (cfg->max_num_batched_tokens > cfg->cap) {
    set_err(res, RS_EINVAL, "max_num_batched_tokens must not exceed cap");
    return res;
  }
  if (cfg->block_size <= 0 || cfg->capacity_blocks <= 0) {
    set_err(res, RS_EINVAL, "block_size and capacity_blocks must be positive");
    return res;
  }
  const int use_dpu = pol >= RS_POLICY_RELSERVE;
  if (use_dpu && !(cfg->tau > 0)) {
    set_err(res, RS_EINVAL, "tau must be positive");
    return res;
  }
  if (!(cfg->noise_sigma >= 0)) {
    set_err(res, RS_EINVAL, "noise_sigma must be non-negative");
    return res;
  }
  int64_t noise_k = 0;
  int noise_ok = 1;
  if (use_dpu && cfg->sample_size < 1) {
    set_err(res, RS_EINVAL, "sample_size must be positive");
    return res;
  }

  eng_t E;
  memset(&E, 0, sizeof E);
  eng_t* e = &E;
  e->tr = tr;
  e->cfg = cfg;
  e->world = world;
  e->pol = policy;
  e->R = R;
  e->N = N;
  e->off = tr->row_off;
  if (rng) e->rng = *rng;

  /* static trie: explicit, or synthesised from the chain/tail structure */
  int64_t* syn_off = NULL;
  int32_t* syn_node = NULL;
  int32_t* syn_parent = NULL;
  int64_t n_nodes = n_nodes_in;
  const int32_t* parent = node_parent_in;
  if (path_off_in && path_node_in) {
    e->path_off = path_off_in;
    e->path_node = path_node_in;
  } else {
    const int64_t B = cfg->block_size;
    syn_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
    int64_t total = 0;
    n_nodes = 0;
    for (int64_t q = 0; q < R; ++q) {
      int64_t P = tr->chain_blocks ? tr->chain_blocks[q] : 0;
      int64_t maxc = 0;
      for (int64_t r = tr->row_off[q]; r < tr->row_off[q + 1]; ++r) {
        int64_t nb = tr->tok[r] / B;
        syn_off[r] = total;
        total += nb;
        int64_t c = nb < P ? nb : P;
        if (c > maxc) maxc = c;
        n_nodes += nb - c;
      }
      n_nodes += maxc;
    }
    syn_off[N] = total;
    syn_node = (int32_t*)malloc(sizeof(int32_t) * (size_t)(total ? total : 1));
    syn_parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_nodes ? n_nodes : 1));
    int64_t next = 0;
    for (int64_t q = 0; q < R; ++q) {
      int64_t P = tr->chain_blocks ? tr->chain_blocks[q] : 0;
      int64_t maxc = 0;
      for (int64_t r = tr->row_off[q]; r < tr->row_off[q + 1]; ++r) {
        int64_t nb = tr->tok[r] / B;
        int64_t c = nb < P ? nb : P;
        if (c > maxc) maxc = c;
      }
      int64_t chain0 = next;
      for (int64_t j = 0; j < maxc; ++j) syn_parent[chain0 + j] = j ? (int32_t)(chain0 + j - 1) : -1;
      next += maxc;
      for (int64_t r = tr->row_off[q]; r < tr->row_off[q + 1]; ++r) {
        int64_t nb = tr->tok[r] / B;
        int64_t c = nb < P ? nb : P;
        for (int64_t j = 0; j < nb; ++j) {
          int32_t id;
          if (j < c) {
            id = (int32_t)(chain0 + j);
          } else {
            id = (int32_t)next++;
            syn_parent[id] = j ? syn_node[syn_off[r] + j - 1] : -1;
          }
          syn_node[syn_off[r] + j] = id;
        }
      }
    }
    e->path_off = syn_off;
    e->path_node = syn_node;
    parent = syn_parent;
  }

  cache_t* c = &e->cache;
  c->B = cfg->block_size;
  c->C = cfg->capacity_blocks;
  c->n_nodes = n_nodes;
  c->parent = parent;
  c->resident = (uint8_t*)calloc((size_t)(n_nodes ? n_nodes : 1), 1);
  c->last_access = (uint64_t*)calloc((size_t)(n_nodes ? n_nodes : 1), sizeof(uint64_t));
  c->nres_child = (int32_t*)calloc((size_t)(n_nodes ? n_nodes : 1), sizeof(int32_t));
  c->pin = (uint32_t*)calloc((size_t)(n_nodes ? n_nodes : 1), sizeof(uint32_t));

  int64_t max_size = 1;
  for (int64_t q = 0; q < R; ++q)
    if (tr->row_off[q + 1] - tr->row_off[q] > max_size) max_size = tr->row_off[q + 1] - tr->row_off[q];
  int64_t scratch = max_size > cfg->max_num_seqs ? max_size : cfg->max_num_seqs;
  if (scratch < cfg->sample_size) scratch = cfg->sample_size;
  e->prefilled = res->prefilled;
  e->gen = res->generated;
  e->prio = res->priority;
  e->completion = res->completion_iter;
  e->live = (uint8_t*)calloc((size_t)(R ? R : 1), 1);
  e->seen_last = (uint8_t*)calloc((size_t)(R ? R : 1), 1);
  e->rec_value = (double*)calloc((size_t)(R ? R : 1), sizeof(double));
  e->new_value = (double*)calloc((size_t)(R ? R : 1), sizeof(double));
  e->new_reused = (uint8_t*)calloc((size_t)(R ? R : 1), 1);
  e->new_override = (uint8_t*)calloc((size_t)(R ? R : 1), 1);
  e->order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(R ? R : 1));
  e->waiting = (wentry*)malloc(sizeof(wentry) * (size_t)(R ? R : 1));
  e->running = (int32_t*)malloc(sizeof(int32_t) * (size_t)(N ? N : 1));
  e->s_utok = (int64_t*)malloc(sizeof(int64_t) * (size_t)scratch);
  e->s_rem = (int32_t*)malloc(sizeof(int32_t) * (size_t)scratch);
  e->s_pre = (uint8_t*)malloc((size_t)scratch);
  e->s_rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)scratch);
  e->s_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)scratch);
  e->s_rels = (int32_t*)malloc(sizeof(int32_t) * (size_t)(N ? N : 1));
  int64_t* relkeys = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cfg->max_num_seqs + 1) * 2);
  int32_t* dec_rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(N ? N : 1));

  /* Engine.__init__: reset + infeasibility check (engine.py:229-239) */
  for (int64_t q = 0; q < R; ++q)
    for (int64_t r = tr->row_off[q]; r < tr->row_off[q + 1]; ++r)
      if ((int64_t)tr->tok[r] + tr->output_limit[q] > cfg->cap) {
        char msg[200];
        snprintf(msg, sizeof msg, "request %lld/%lld needs %lld KV tokens > cap %lld",
                 (long long)tr->rel_id[q], (long long)(r - tr->row_off[q]),
                 (long long)tr->tok[r] + tr->output_limit[q], (long long)cfg->cap);
        set_err(res, RS_EINFEASIBLE, msg);
        goto cleanup;
      }
  for (int32_t q = 0; q < R; ++q) e->order[q] = q;
  g_sort_eng = e;
  qsort(e->order, (size_t)R, sizeof(int32_t), cmp_arrival); /* engine.py:211-213 */

  const int force_prefill = pol == RS_POLICY_RELSERVE_PP, force_decode = pol == RS_POLICY_RELSERVE_DP;
  const int prefill_first = pol == RS_POLICY_FCFS || pol == RS_POLICY_SP;
  int64_t log_cap = 0, dpuoff_cap = 0, waitoff_cap = 0, wait_cap = 0, rngcap = 0, iw_cap = 0;
  const double t_start = now_s();
  res->status = RS_OK;

  while (e->n_live > 0 || e->next_arrival < R) {
    if (e->iteration >= cfg->iteration_limit) {
      char msg[128];
      snprintf(msg, sizeof msg, "iteration limit %lld exceeded", (long long)cfg->iteration_limit);
      set_err(res, RS_EABORT_LIMIT, msg);
      break;
    }
    const double t_iter = now_s();
    /* admit_arrivals (engine.py:243-269) */
    while (e->next_arrival < R && tr->arrival[e->order[e->next_arrival]] <= e->clock) {
      int32_t rq = e->order[e->next_arrival++];
      e->waiting[e->n_waiting].rq = rq;
      e->waiting[e->n_waiting].pend = 0;
      e->n_waiting++;
      e->live[rq] = 1;
      e->n_live++;
      double p = 0.0;
      if (pol == RS_POLICY_SP) p = tr->static_prio ? tr->static_prio[rq] : 0.0;
      if (pol == RS_POLICY_SP || pol == RS_POLICY_FCFS)
        for (int64_t r = tr->row_off[rq]; r < tr->row_off[rq + 1]; ++r) e->prio[r] = p;
    }
    /* _update_priorities (engine.py:277-281) */
    double t0 = now_s();
    int64_t n_est = 0;
    if (rec_flags & OR_REC_DPU) {
      if (grow((void**)&res->dpu_off, &dpuoff_cap, e->iteration + 2, sizeof(int64_t))) goto oom;
      res->dpu_off[e->iteration] = res->n_dpu;
    }
    if (use_dpu) {
      int rc = dpu_update(e, &n_est, rec_flags, res);
      if (rc) {
        set_err(res, rc, rc == RS_EINFEASIBLE ? "uncached tokens exceed cap" : "dpu failure");
        break;
      }
    }
    {
      int64_t w = 0;
      for (int64_t i = 0; i < e->n_waiting; ++i) {
        int32_t rq = e->waiting[i].rq;
        if (e->waiting[i].pend < tr->row_off[rq + 1] - tr->row_off[rq]) e->waiting[w++] = e->waiting[i];
      }
      e->n_waiting = w;
      qsort(e->waiting, (size_t)w, sizeof(wentry), cmp_waiting);
    }
    const double t_dpu = now_s() - t0;
    res->dpu_wall_s += t_dpu;
    if (rec_flags & OR_REC_WAITING) {
      if (grow((void**)&res->wait_off, &waitoff_cap, e->iteration + 2, sizeof(int64_t))) goto oom;
      res->wait_off[e->iteration] = res->n_wait;
      if (grow((void**)&res->wait, &wait_cap, res->n_wait + e->n_waiting, sizeof(int32_t))) goto oom;
      for (int64_t i = 0; i < e->n_waiting; ++i) res->wait[res->n_wait++] = e->waiting[i].rq;
    }
    if (rec_flags & OR_REC_RNG) {
      if (grow((void**)&res->rng_trace, &rngcap, 4 * (e->iteration + 1), sizeof(uint64_t))) goto oom;
      uint64_t* q = res->rng_trace + 4 * e->iteration;
      q[0] = e->rng.state_hi;
      q[1] = e->rng.state_lo;
      q[2] = e->rng.has_uint32;
      q[3] = e->rng.uinteger;
    }

    /* _build_candidates (engine.py:285-308) */
    t0 = now_s();
    const int64_t mns = cfg->max_num_seqs;
    int64_t nd = e->n_running;
    const int32_t* dec = e->running;
    if (nd > mns) { /* build_decode_candidate truncation (arranger.py:71-77); dead in Engine */
      memcpy(dec_rows, e->running, sizeof(int32_t) * (size_t)nd);
      /* sort by (arrival, rel_id, req_id): rows are stored in trace order, and trace
         order is (arrival, then list order); use a stable insertion sort on keys */
      for (int64_t i = 1; i < nd; ++i) {
        int32_t x = dec_rows[i];
        int64_t j = i - 1;
        while (j >= 0) {
          int32_t y = dec_rows[j];
          int32_t qx = 0, qy = 0;
          /* locate relQueries by binary search over row_off */
          int64_t lo = 0, hi = R;
          while (hi - lo > 1) { int64_t m = (lo + hi) / 2; if (tr->row_off[m] <= x) lo = m; else hi = m; }
          qx = (int32_t)lo;
          lo = 0; hi = R;
          while (hi - lo > 1) { int64_t m = (lo + hi) / 2; if (tr->row_off[m] <= y) lo = m; else hi = m; }
          qy = (int32_t)lo;
          double ax = tr->arrival[qx], ay = tr->arrival[qy];
          int gt = ay > ax || (ay == ax && (tr->rel_id[qy] > tr->rel_id[qx] ||
                   (tr->rel_id[qy] == tr->rel_id[qx] && (y - tr->row_off[qy]) > (x - tr->row_off[qx]))));
          if (!gt) break;
          dec_rows[j + 1] = y;
          j--;
        }
        dec_rows[j + 1] = x;
      }
      nd = mns;
      dec = dec_rows;
    }
    int32_t head_rq = e->n_waiting ? e->waiting[0].rq : -1;
    int64_t head_pend = e->n_waiting ? e->waiting[0].pend : 0;
    int64_t taken = 0, utok_sum = 0;
    if (head_rq >= 0) { /* build_prefill_candidate (arranger.py:80-112) */
      int64_t kv_need = 0;
      const int64_t headroom = cfg->cap - e->kv_reserved;
      for (int64_t r = tr->row_off[head_rq] + head_pend; r < tr->row_off[head_rq + 1]; ++r) {
        int64_t utok = cache_match(&e->cache, row_path(e, r), row_nb(e, r), tr->tok[r], 0, 0);
        int64_t kv = (int64_t)tr->tok[r] + tr->output_limit[head_rq];
        if (taken && utok_sum + utok > cfg->max_num_batched_tokens) break;
        if (e->n_running + taken + 1 > mns) break;
        if (kv_need + kv > headroom) break;
        taken++;
        utok_sum += utok;
        kv_need += kv;
      }
    }
    const int has_p = taken > 0, has_d = nd > 0;
    double m_plus = NAN, m_minus = NAN;
    int64_t dmin_pos = -1;
    if (has_d) {
      m_plus = e->prio[dec[0]];
      dmin_pos = 0;
      for (int64_t i = 1; i < nd; ++i)
        if (e->prio[dec[i]] < m_plus) {
          m_plus = e->prio[dec[i]];
          dmin_pos = i;
        }
    }
    const int64_t pfirst = has_p ? tr->row_off[head_rq] + head_pend : -1;
    if (has_p) {
      m_minus = e->prio[pfirst];
      for (int64_t i = 1; i < taken; ++i)
        if (e->prio[pfirst + i] < m_minus) m_minus = e->prio[pfirst + i];
    }
    int action, kase;
    double dp = NAN, dm = NAN, dt = NAN, out_mp = m_plus, out_mm = m_minus;
    if (prefill_first) { /* engine.py:387-395 */
      kase = RS_CASE_FORCED;
      if (has_p) action = RS_ACTION_PREFILL;
      else if (has_d) action = RS_ACTION_DECODE;
      else {
        action = RS_ACTION_IDLE;
        out_mp = out_mm = NAN;
      }
    } else {
      int have_proj = 0;
      if (has_p && has_d && m_plus <= m_minus) { /* engine.py:397-415 + project_delta (arranger.py:115-143) */
        int64_t nrel = 0;
        for (int64_t i = 0; i < nd; ++i) {
          int64_t lo = 0, hi = R, x = dec[i];
          while (hi - lo > 1) { int64_t m = (lo + hi) / 2; if (tr->row_off[m] <= x) lo = m; else hi = m; }
          relkeys[2 * nrel] = tr->rel_id[lo];
          relkeys[2 * nrel + 1] = lo;
          nrel++;
        }
        /* sorted(set(rel_ids)) */
        int64_t* keys = relkeys;
        for (int64_t i = 1; i < nrel; ++i) { /* insertion sort of (rel_id, rq) pairs by rel_id */
          int64_t k0 = keys[2 * i], k1 = keys[2 * i + 1];
          int64_t j = i - 1;
          while (j >= 0 && keys[2 * j] > k0) {
            keys[2 * j + 2] = keys[2 * j];
            keys[2 * j + 3] = keys[2 * j + 1];
            j--;
          }
          keys[2 * j + 2] = k0;
          keys[2 * j + 3] = k1;
        }
        int64_t u = 0;
        for (int64_t i = 0; i < nrel; ++i)
          if (u == 0 || keys[2 * (u - 1)] != keys[2 * i]) {
            keys[2 * u] = keys[2 * i];
            keys[2 * u + 1] = keys[2 * i + 1];
            u++;
          }
        const rs_cost_model* m = policy;
        double l_prefill = m->alpha_p * (double)utok_sum + m->beta_p;
        int64_t ol_p = tr->output_limit[head_rq];
        double delta_plus = l_prefill * (double)u;
        int64_t max_ol = 0;
        for (int64_t i = 0; i < u; ++i) {
          int64_t ol = tr->output_limit[keys[2 * i + 1]];
          int64_t mn = ol < ol_p ? ol : ol_p;
          delta_plus += m->alpha_d * (double)taken * (double)mn;
          if (ol > max_ol) max_ol = ol;
        }
        int64_t mn = ol_p < max_ol ? ol_p : max_ol;
        double delta_minus = -((double)e->n_waiting * m->beta_d * (double)mn);
        dp = delta_plus;
        dm = delta_minus;
        dt = delta_plus + delta_minus;
        have_proj = 1;
      }
      /* decide_next (arranger.py:146-179) */
      if (!has_p && !has_d) {
        action = RS_ACTION_IDLE;
        kase = RS_CASE_FORCED;
        out_mp = out_mm = NAN;
      } else if (!has_d) {
        action = RS_ACTION_PREFILL;
        kase = RS_CASE_FORCED;
      } else if (!has_p) {
        action = RS_ACTION_DECODE;
        kase = RS_CASE_FORCED;
      } else {
        int64_t lo = 0, hi = R, x = dec[dmin_pos];
        while (hi - lo > 1) { int64_t mm = (lo + hi) / 2; if (tr->row_off[mm] <= x) lo = mm; else hi = mm; }
        if (tr->rel_id[lo] == tr->rel_id[head_rq]) {
          action = RS_ACTION_PREFILL;
          kase = RS_CASE_INTERNAL;
        } else if (m_plus > m_minus) {
          action = RS_ACTION_PREFILL;
          kase = RS_CASE_PREEMPT;
        } else {
          kase = RS_CASE_TRANSITIONAL;
          if (force_prefill) action = RS_ACTION_PREFILL;
          else if (force_decode) action = RS_ACTION_DECODE;
          else if (have_proj && dt < 0) action = RS_ACTION_PREFILL;
          else action = RS_ACTION_DECODE;
        }
      }
      if (!(kase == RS_CASE_TRANSITIONAL)) dp = dm = dt = NAN; /* only transitional decisions carry the projection */
    }
    res->aba_wall_s += now_s() - t0;

    /* decision record */
    if (grow((void**)&res->log, &log_cap, e->iteration + 1, sizeof(rs_iter_record))) goto oom;
    rs_iter_record* rec = &res->log[e->iteration];
    memset(rec, 0, sizeof *rec);
    rec->iteration = e->iteration;
    rec->clock = e->clock;
    rec->m_plus = out_mp;
    rec->m_minus = out_mm;
    rec->delta_plus = dp;
    rec->delta_minus = dm;
    rec->delta_total = dt;
    rec->action = action;
    rec->kase = kase;
    rec->head = head_rq;
    rec->n_waiting = (int32_t)e->n_waiting;
    rec->batch_rq = -1;
    rec->n_reestimated = (int32_t)n_est;

    if (action == RS_ACTION_PREFILL) { /* _execute_prefill (engine.py:315-341) */
      const double start = e->clock;
      int64_t ut = 0;
      for (int64_t i = 0; i < taken; ++i) {
        int64_t r = pfirst + i;
        ut += cache_match(&e->cache, row_path(e, r), row_nb(e, r), tr->tok[r], 1, 1);
        int rc = cache_insert(&e->cache, row_path(e, r), row_nb(e, r));
        if (rc) {
          set_err(res, rc, "prefix cache cannot evict: all resident blocks pinned");
          goto done_loop;
        }
      }
      double duration = world_duration(cfg, noise, noise_len, &noise_k, world->alpha_p * (double)ut + world->beta_p,
                                       &noise_ok);
      if (!noise_ok) {
        set_err(res, RS_EINVAL, "noise sequence shorter than the executed batches");
        goto done_loop;
      }
      for (int64_t i = 0; i < taken; ++i) {
        int64_t r = pfirst + i;
        e->prefilled[r] = 1;
        e->running[e->n_running++] = (int32_t)r;
        e->kv_reserved += (int64_t)tr->tok[r] + tr->output_limit[head_rq];
      }
      e->waiting[0].pend += taken;
      if (e->waiting[0].pend == tr->row_off[head_rq + 1] - tr->row_off[head_rq]) {
        memmove(e->waiting, e->waiting + 1, sizeof(wentry) * (size_t)(e->n_waiting - 1));
        e->n_waiting--;
      }
      e->clock += duration;
      if (isnan(res->first_prefill_start[head_rq])) res->first_prefill_start[head_rq] = start;
      res->last_prefill_end[head_rq] = e->clock;
      rec->batch_rq = head_rq;
      rec->batch_first = (int32_t)head_pend;
      rec->batch_n = (int32_t)taken;
    } else if (action == RS_ACTION_DECODE) { /* _execute_decode (engine.py:343-363) */
      double duration = world_duration(cfg, noise, noise_len, &noise_k, world->alpha_d * (double)nd + world->beta_d,
                                       &noise_ok);
      if (!noise_ok) {
        set_err(res, RS_EINVAL, "noise sequence shorter than the executed batches");
        goto done_loop;
      }
      e->clock += duration;
      int64_t nfin = 0, ndone = 0;
      for (int64_t i = 0; i < nd; ++i) {
        int32_t r = dec[i];
        e->gen[r] += 1;
        if (row_done(e, r)) {
          ndone++;
          e->completion[r] = e->iteration;
          int64_t lo = 0, hi = R;
          while (hi - lo > 1) { int64_t m = (lo + hi) / 2; if (tr->row_off[m] <= r) lo = m; else hi = m; }
          e->kv_reserved -= (int64_t)tr->tok[r] + tr->output_limit[lo];
          int all = 1;
          for (int64_t x = tr->row_off[lo]; x < tr->row_off[lo + 1]; ++x)
            if (!row_done(e, x)) {
              all = 0;
              break;
            }
          if (all) {
            int dup = 0;
            for (int64_t f = 0; f < nfin; ++f)
              if (e->s_rels[f] == lo) dup = 1;
            if (!dup) e->s_rels[nfin++] = (int32_t)lo;
          }
        }
      }
      if (ndone) {
        int64_t w = 0;
        for (int64_t i = 0; i < e->n_running; ++i)
          if (!row_done(e, e->running[i])) e->running[w++] = e->running[i];
        e->n_running = w;
      }
      for (int64_t f = 0; f < nfin; ++f) {
        int32_t q = e->s_rels[f];
        res->last_decode_end[q] = e->clock;
        e->live[q] = 0;
        e->n_live--;
      }
      rec->batch_n = (int32_t)nd;
    } else { /* idle (engine.py:439-447) */
      if (e->next_arrival >= R) {
        if (e->n_live) {
          set_err(res, RS_EABORT_IDLE, "engine idle with live relQueries and no future arrivals");
          rec->kv_reserved = e->kv_reserved;
          res->n_log = e->iteration + 1;
          goto done_loop;
        }
        rec->kv_reserved = e->kv_reserved;
        res->n_log = e->iteration + 1;
        goto done_loop; /* break without incrementing (engine.py:446) */
      }
      double nxt = tr->arrival[e->order[e->next_arrival]];
      if (nxt > e->clock) e->clock = nxt;
    }
    rec->kv_reserved = e->kv_reserved;
    if (grow((void**)&res->iter_wall, &iw_cap, e->iteration + 1, sizeof(double))) goto oom;
    double w_it = now_s() - t_iter;
    res->iter_wall[e->iteration] = w_it;
    if (n_est > 0 && w_it > res->first_sight_wall_s) {
      res->first_sight_wall_s = w_it;
      res->first_sight_iter = e->iteration;
    }
    e->iteration += 1;
    res->n_log = e->iteration;
  }
done_loop:
  if (rec_flags & OR_REC_DPU && res->dpu_off) res->dpu_off[res->n_log] = res->n_dpu;
  if (rec_flags & OR_REC_WAITING && res->wait_off) res->wait_off[res->n_log] = res->n_wait;
  res->total_wall_s = now_s() - t_start;
  res->iterations = e->iteration;
  res->clock = e->clock;
  res->cache_hit_tokens = c->hit_total;
  res->cache_miss_tokens = c->miss_total;
  res->kv_reserved = e->kv_reserved;
  res->rng = e->rng;
  goto cleanup;
oom:
  set_err(res, RS_ENOMEM, "out of memory");
cleanup:
  free(e->live); free(e->seen_last); free(e->rec_value); free(e->new_value); free(e->new_reused);
  free(e->new_override); free(e->order); free(e->waiting); free(e->running); free(e->s_utok);
  free(e->s_rem); free(e->s_pre); free(e->s_rows); free(e->s_idx); free(e->s_rels);
  free(relkeys); free(dec_rows);
  free(c->resident); free(c->last_access); free(c->nres_child); free(c->pin); free(c->heap);
  free(c->skipped);
  free(syn_off); free(syn_node); free(syn_parent);
  return res;
}

void or_free(or_result* r) {
  if (!r) return;
  free(r->log); free(r->first_prefill_start); free(r->last_prefill_end); free(r->last_decode_end);
  free(r->generated); free(r->prefilled); free(r->completion_iter); free(r->priority);
  free(r->dpu_off); free(r->dpu); free(r->wait_off); free(r->wait); free(r->rng_trace);
  free(r->iter_wall);
  free(r);
}
