// cache_model.cuh -- the reference prefix cache (trie + lazy LRU heap,
// prefix_cache.py:41-138) as used by the engine, reduced to per-relQuery /
// per-row counters.
//
// For traces whose block trie is a forest of one shared chain per relQuery
// plus private per-row tails (generate_trace / load_trace traces; checked on
// the host for explicit token lists):
//   * a relQuery's resident chain is a prefix of length m, touched as one
//     consecutive run of the global touch clock starting at c0 (every touch
//     of a chain block is part of a match+insert of one of its rows);
//   * a row's tail is touched only when the row is prefilled, so tails enter
//     the FIFO in touch order and each one's leaf time is t0 + tres - 1;
//   * eviction takes the minimum-time unpinned leaf (the lazy heap pops in
//     (last_access, id) order, skips stale / non-leaf / pinned entries and
//     re-pushes the skipped ones): either the FIFO head's last block or the
//     last block of the oldest chain that has no resident tail (cc list).
//     Evicting a leaf exposes its parent, which is older than every other
//     leaf, so a unit is always drained consecutively.
// DESIGN.md "Prefix-cache model" has the full argument.
#pragma once
#include "engine_state.cuh"

namespace rsd {

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

// Evict k blocks from the end of the chain candidate at the front.
__device__ __forceinline__ void cc_evict_front(Ctl& c, const RqView& rq, long long k) {
  CcEnt& e = c.cc[0];
  e.m -= (int)k;
  e.key -= (unsigned long long)k;
  rq.m[e.rank] = e.m;
  c.count -= k;
  if (e.m == 0) {
    for (int i = 1; i < c.cc_n; ++i) c.cc[i - 1] = c.cc[i];
    c.cc_n--;
  }
}

// Exact single-thread eviction until count <= C; cur_rank / cur_tail identify
// the pinned path (prefix_cache.py:107-120): the inserted row's chain and, if
// it has one, its tail (the FIFO back).
__device__ int cache_evict(Ctl& c, const TraceDev& T, const RqView& rq, long long C, int cur_rank,
                           bool cur_tail) {
  while (c.count > C) {
    const bool have_f = c.fifo_head < c.fifo_tail;
    unsigned long long kf = ~0ULL, kc = ~0ULL;
    FifoEnt fe;
    if (have_f) {
      fe = T.fifo[c.fifo_head & (T.fifo_cap - 1)];
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
        const int nt = rq.ntails[a] - 1;
        rq.ntails[a] = nt;
        const int mm = rq.m[a];
        if (nt == 0 && mm > 0 && !cc_insert(c, rq.c0[a] + (unsigned long long)(mm - 1), a, mm))
          return RS_EUNSUPPORTED;
      } else {
        T.fifo[c.fifo_head & (T.fifo_cap - 1)].tres = fe.tres;
      }
    } else {
      if (c.cc[0].rank == cur_rank) return RS_ECACHE_PINNED;
      const long long k = need < c.cc[0].m ? need : c.cc[0].m;
      cc_evict_front(c, rq, k);
    }
  }
  return RS_OK;
}

// Exact path for one row: match_uncached(refresh=True, record=True) then
// insert (engine.py:321-323).  Returns the row's uncached tokens, or -1 on
// error (status set).  Single thread.
__device__ long long prefill_row_cache(Ctl& c, const TraceDev& T, const RqView& rq, const Params& P, int a,
                                       int tok) {
  const long long B = P.cfg.block_size;
  const long long C = P.cfg.capacity_blocks;
  // a sequence longer than the whole cache inserts only its first C blocks
  // (prefix_cache.py:101-103, last_insert_truncated)
  const int nb = (int)(tok / B < C ? tok / B : C);
  const int Pc = rq.chain[a] < nb ? rq.chain[a] : nb;
  const int T_len = nb - Pc;
  const int mb = rq.m[a];
  const long long hit = B * mb;
  cc_remove(c, a);  // the chain is touched again
  c.hit += hit;
  c.miss += tok - hit;
  c.tclock += (unsigned long long)mb;  // match touches the resident chain
  const unsigned long long c0 = c.tclock + 1;
  c.tclock += (unsigned long long)Pc;  // insert touches the whole chain
  const unsigned long long t0 = c.tclock + 1;
  c.tclock += (unsigned long long)T_len;  // ... then the private tail
  c.count += (long long)(Pc - mb) + T_len;
  rq.m[a] = Pc;
  rq.c0[a] = c0;
  if (T_len > 0) {
    FifoEnt e;
    e.t0 = t0;
    e.rank = a;
    e.tres = T_len;
    T.fifo[c.fifo_tail & (T.fifo_cap - 1)] = e;
    c.fifo_tail++;
    rq.ntails[a] += 1;
  } else if (Pc > 0 && rq.ntails[a] == 0) {
    if (!cc_insert(c, c0 + (unsigned long long)(Pc - 1), a, Pc)) {
      c.status = RS_EUNSUPPORTED;
      c.error_detail = 1;
      return -1;
    }
  }
  const int rc = cache_evict(c, T, rq, P.cfg.capacity_blocks, a, T_len > 0);
  if (rc) {
    c.status = rc;
    c.error_detail = 2;
    return -1;
  }
  return tok - hit;
}

// Sequential drain of E blocks in LRU order from the staged FIFO head and the
// chain candidates (thread 0; the cold path of prefill_fast when chain
// candidates are pending or the parallel drain's preconditions fail).
__device__ void drain_sequential(Shared& S, const TraceDev& T, long long E, int Wn, long long head0) {
  Ctl& c = S.c;
  const RqView& rq = S.rq;
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
      cc_evict_front(c, rq, k);
    }
  }
  if (!ok) {
    c.status = RS_ECACHE_PINNED;
    c.error_detail = 4;
  }
  if (j < Wn) T.fifo[(head0 + j) & (T.fifo_cap - 1)].tres = S.win.tres[j];
  S.fp_popped = j;
  c.fifo_head = head0 + j;
}

// Batched prefill advance (all threads).  Every row of a prefill batch
// belongs to the head relQuery h, whose chain is pinned by each row's insert
// and fully resident after the first one.  When every row also has a private
// tail, the reference's per-row insert/evict interleaving evicts, in LRU
// order, exactly the first E = max(0, count + new - C) blocks of the
// pre-batch resident set -- whatever the interleaving, as long as E does not
// exceed those blocks.  So the per-row touch times and FIFO pushes come from
// prefix sums, and one thread then drains E blocks from the FIFO head (staged
// in shared memory) and the chain candidates.  Returns false (nothing
// changed) when the preconditions fail; the caller then runs the exact
// per-row path.  tokv: the batch rows' tok (staged by the candidate scan).
// G: the executing warp group (the whole CTA, or group M of the pipelined
// iteration); kHand: group M waits at the handoff barrier before its first
// write of state group D reads (rq.m in the drain) -- only when returning true.
template <bool kC, class G = GAll, bool kHand = false>
__device__ bool prefill_fast(const Params& P, const TraceDev& T, Shared& S, int h, int n, const int* tokv,
                             long long& ut_out) {
  Ctl& c = S.c;
  const RqView rq = S.rq;  // by value: the table pointers stay in registers across the barriers
  const int tid = threadIdx.x;
  const long long B = kC ? 16 : P.cfg.block_size;  // kC: the default block size (engine.py:152)
  const long long C = P.cfg.capacity_blocks;
  const int Pc = rq.chain[h];
  const int m0 = rq.m[h];
  const unsigned long long tc = c.tclock;
  const long long head0 = c.fifo_head, tail0 = c.fifo_tail, count0 = c.count;
  // 1. per-row tail blocks: prefix sums of (tail, tok, tail-less rows) in one scan
  long long Tv[kMaxRun / G::kN], inclT[kMaxRun / G::kN];
  long long cT = 0, cTok = 0;
  int n_bad = 0;
#pragma unroll
  for (int s = 0; s < kMaxRun / G::kN; ++s) {
    Tv[s] = 0;
    inclT[s] = 0;
    if (s * G::kN < n) {
      const int i = s * G::kN + tid;
      int tk = 0, tl = 0;
      if (i < n) {
        tk = tokv[i];
        tl = (int)(tk / B) - Pc;
      }
      // rows without a private tail, or truncated by the capacity: the exact path
      int v[3] = {tl, tk, (i < n && (tl <= 0 || tk / B > C)) ? 1 : 0}, tot[3];
      group_scan32<G, 3>(v, S.s32, tot, tid >> 5);
      Tv[s] = tl;
      inclT[s] = cT + v[0];
      cT += tot[0];
      cTok += tot[1];
      n_bad += tot[2];
    }
  }
  const long long newn = (long long)(Pc - m0) + cT;
  const long long E = count0 + newn > C ? count0 + newn - C : 0;
  const long long n_old = tail0 - head0;
  const int Wn = (int)(E < n_old ? E : n_old);
  if (n_bad || E > count0 - m0 || Wn > kWin) return false;  // block-uniform
  phase_mark(c, 13);
  // 2. FIFO pushes: row i's chain / tail touch times from prefix sums of touches
#pragma unroll
  for (int s = 0; s < kMaxRun / G::kN; ++s) {
    const int i = s * G::kN + tid;
    if (i < n) {
      const long long before =
          i == 0 ? 0 : (long long)m0 + (long long)(i - 1) * Pc + (long long)i * Pc + (inclT[s] - Tv[s]);
      const long long mb = i == 0 ? m0 : Pc;
      const unsigned long long c0i = tc + (unsigned long long)(before + mb + 1);
      FifoEnt e;
      e.t0 = c0i + (unsigned long long)Pc;
      e.rank = h;
      e.tres = (int)Tv[s];
      T.fifo[(tail0 + i) & (T.fifo_cap - 1)] = e;
      if (i == n - 1) S.fp_c0_last = c0i;
    }
  }
  //    stage the FIFO head (the oldest tails) and their relQueries' chain state;
  //    thread 0 meanwhile drops h from the chain candidates (its chain is touched)
  for (int j = tid; j < Wn; j += G::kN) {
    const FifoEnt e = T.fifo[(head0 + j) & (T.fifo_cap - 1)];
    S.win.t0[j] = e.t0;
    S.win.rank[j] = e.rank;
    S.win.tres[j] = e.tres;
    S.win.mm[j] = rq.m[e.rank];
    S.win.c0[j] = rq.c0[e.rank];
    atomicAdd(&rq.scr_cnt[e.rank], 1);
    atomicMax(&rq.scr_last[e.rank], j);
  }
  if (tid == 0) {
    c.alg_bytes += 16LL * Wn;  // staged FIFO head
    cc_remove(c, h);
    S.fp_par = c.cc_n == 0;
    S.fp_cut = 0x7FFFFFFF;
  }
  G::sync();
  phase_mark(c, 14);
  if constexpr (kHand) handoff_wait();  // group D has read the chain lengths (rq.m) it uses
  // 3. Parallel drain (no chain candidate pending): in LRU order the FIFO units
  // are consumed front to back, each relQuery's chain right after its last
  // tail -- provided that chain is older than the next unit's leaf.  Blocks
  // per unit b_j = tres_j (+ m_j if it is the relQuery's last resident tail);
  // the cut is the first unit whose inclusive sum reaches E.  The thread of
  // unit j computes its `last` flag itself, so no barrier separates them.
  bool par = S.fp_par;
  if (par && E > 0) {
    long long carry = 0;
    for (int base = 0; base < Wn; base += G::kN) {
      const int j = base + tid;
      int bj = 0;
      if (j < Wn) {
        const int a = S.win.rank[j];
        const int last = (a != h && rq.scr_last[a] == j && rq.scr_cnt[a] == rq.ntails[a]) ? 1 : 0;
        S.win.last[j] = last;
        bj = S.win.tres[j] + (last ? S.win.mm[j] : 0);
      }
      int v[1] = {bj}, tot[1];
      group_scan32<G, 1>(v, S.s32, tot, tid >> 5);
      if (j < Wn && carry + v[0] >= E && carry + v[0] - bj < E) {  // the unique cut unit
        S.fp_cut = j;
        S.fp_rem = E - (carry + v[0] - bj);
      }
      carry += tot[0];
    }
    G::sync();
    const int cut = S.fp_cut;
    if (cut == 0x7FFFFFFF) {
      par = false;
    } else {
      const long long rem_cut = S.fp_rem;
      bool bad = false;
      for (int j = tid; j <= cut && j < Wn; j += G::kN) {
        const bool chain_evicted = S.win.last[j] && (j < cut || rem_cut > S.win.tres[j]);
        if (chain_evicted) {
          const unsigned long long kc = S.win.c0[j] + (unsigned long long)(S.win.mm[j] - 1);
          const bool next_in = j + 1 < Wn;
          const unsigned long long kn = next_in ? S.win.t0[j + 1] + (unsigned long long)(S.win.tres[j + 1] - 1) : ~0ULL;
          if ((!next_in && j + 1 < n_old) || !(kc < kn)) bad = true;
        }
      }
      par = !G::sync_or(bad);
      if (par) {
        for (int j = tid; j < cut; j += G::kN) {
          atomicSub(&rq.ntails[S.win.rank[j]], 1);
          if (S.win.last[j]) rq.m[S.win.rank[j]] = 0;
        }
        if (tid == 0) {
          const int a = S.win.rank[cut];
          const int tr = S.win.tres[cut];
          int head_adv = cut;
          if (rem_cut < tr) {
            T.fifo[(head0 + cut) & (T.fifo_cap - 1)].tres = tr - (int)rem_cut;
          } else {
            head_adv = cut + 1;
            atomicSub(&rq.ntails[a], 1);
            if (S.win.last[cut]) {
              const int mm = S.win.mm[cut] - (int)(rem_cut - tr);
              rq.m[a] = mm;
              if (mm > 0 && !cc_insert(c, S.win.c0[cut] + (unsigned long long)(mm - 1), a, mm)) {
                c.status = RS_EUNSUPPORTED;
                c.error_detail = 5;
              }
            }
          }
          c.count -= E;
          c.fifo_head = head0 + head_adv;
        }
      }
    }
  } else if (par && tid == 0) {
    c.fifo_head = head0;
  }
  // 4. sequential drain (cold path) and the batch's own bookkeeping (thread 0);
  //    h's tail count is updated atomically: drain threads may be retiring h's older tails
  if (!par) {
    if (tid == 0) {
      // the last flags for the sequential drain (the parallel branch computed them itself)
      for (int j = 0; j < Wn; ++j) {
        const int a = S.win.rank[j];
        S.win.last[j] = (a != h && rq.scr_last[a] == j && rq.scr_cnt[a] == rq.ntails[a]) ? 1 : 0;
      }
      drain_sequential(S, T, E, Wn, head0);
    }
    G::sync();
  }
  if (tid == 0) {
    const long long hitb = (long long)m0 + (long long)(n - 1) * Pc;
    c.hit += B * hitb;
    c.miss += cTok - B * hitb;
    ut_out = cTok - B * hitb;
    c.tclock = tc + (unsigned long long)(hitb + (long long)n * Pc + cT);
    c.count += newn;
    c.fifo_tail = tail0 + n;
    rq.m[h] = Pc;
    rq.c0[h] = S.fp_c0_last;
    atomicAdd(&rq.ntails[h], n);
  }
  // 5. reset the staging counters; the sequential drain's popped units lose a tail
  const int popped = par ? 0 : S.fp_popped;
  for (int j = tid; j < Wn; j += G::kN) {
    const int a = S.win.rank[j];
    if (j < popped) atomicSub(&rq.ntails[a], 1);
    rq.scr_cnt[a] = 0;
    rq.scr_last[a] = -1;
  }
  return true;  // the caller's next barrier orders these writes
}

}  // namespace rsd
