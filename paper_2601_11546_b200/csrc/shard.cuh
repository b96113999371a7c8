// shard.cuh -- the sharded pool (BASELINE config 5): one trace,
// its relQueries owned round-robin by admission rank across `world` shards.
//
// Every shard keeps a replica of the whole scheduler state (clock, queues,
// running list, prefix-cache model, RNG, per-relQuery counters) and replays
// the identical arranger and state advance, so replicas never diverge.  What
// is sharded is the per-iteration estimation work: a shard re-estimates only
// the partially prefilled relQueries it owns (dpu.cuh, `own`) and orders only
// its own waiting relQueries.  Once per iteration the shards exchange one
// record each -- their local waiting head and the priorities they computed --
// and every shard then knows the global head (min over shards of
// (priority bits, rank), the reference's (priority, arrival, rel_id) order,
// engine.py:175-176) and every priority the arranger reads.
//
// The exchange is done inside the persistent kernel over peer memory (an
// allgather of fixed-size records): a shard stores its record into every
// peer's mailbox (NVLink P2P stores on a multi-GPU box, where the mailboxes are
// CUDA-IPC mapped; plain global stores between the CTAs of one launch when all
// shards run on one GPU) and reads its own mailbox.  The record travels as
// 8-byte words that each carry 32 data bits and a 32-bit flag (the iteration
// + 1): an aligned 8-byte store is single-copy atomic, so a reader that sees
// the flag sees the data (the "LL" protocol of NCCL), and neither side needs
// a memory fence -- a fence or acquire would also invalidate the SM's L1 and
// make the rest of the iteration re-fetch its working set.  Records are
// double-buffered by iteration parity: a shard can only reach iteration t+2
// after every shard published t+1, which each does only after consuming t's.
#pragma once
#include "engine_state.cuh"

namespace rsd {

// One shard's record for one iteration, as flagged words (flag << 32 | data):
// w[0], w[1] local waiting head key (priority bits, lo / hi), w[2] its rank,
// w[3 + 2j], w[4 + 2j] the priority of act-list position j (lo / hi) for the
// positions whose relQuery the sender owns.
struct alignas(16) ShardRec {
  unsigned long long w[3 + 2 * kMaxAct];
};

// A shard's mailbox: ShardRec[world][2] (sender, iteration parity).
__host__ __device__ inline size_t mailbox_bytes(int world) { return sizeof(ShardRec) * 2 * (size_t)world; }

__device__ __forceinline__ void ll_store(unsigned long long* p, unsigned flag, unsigned data) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(((unsigned long long)flag << 32) | data)
               : "memory");
}

// Spin until the word carries `flag`; false after ~35 s (a peer never arrived).
__device__ __forceinline__ bool ll_load(const unsigned long long* p, unsigned flag, unsigned& data) {
  long long t0 = 0;
  for (int spins = 0;; ++spins) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if ((unsigned)(v >> 32) == flag) {
      data = (unsigned)v;
      return true;
    }
    if (spins == 0) t0 = clock64();
    else if (clock64() - t0 > (1LL << 36)) return false;  // ~35 s: a peer is gone
  }
}

// All threads.  In: this shard's local head (key, idx), its owned priorities in
// rq.prio (written before the DPU's closing barrier).  Out: the global head in
// (key, idx); every owned-elsewhere priority of the act list written into this
// replica's rq.prio.  Returns false on an exchange timeout (status set).
__device__ bool shard_exchange(const TraceDev& T, Shared& S, unsigned long long& key, int& idx) {
  Ctl& c = S.c;
  const RqView& rq = S.rq;
  const int W = T.shard_world, me = T.shard_rank;
  const int tid = threadIdx.x;
  const unsigned flag = (unsigned)(c.iteration + 1);
  const int par = (int)(c.iteration & 1);
  const int n_act = c.n_act;
  // 1. publish: header to every peer (thread d), owned priorities (thread j)
  if (tid < W && tid != me) {
    unsigned long long* w = T.peers[tid][2 * me + par].w;
    ll_store(w + 0, flag, (unsigned)key);
    ll_store(w + 1, flag, (unsigned)(key >> 32));
    ll_store(w + 2, flag, (unsigned)idx);
  }
  for (int j = tid; j < n_act; j += kThreads) {
    const int a = c.act[j];
    if (a % W == me) {
      const unsigned long long v = (unsigned long long)__double_as_longlong(rq.prio[a]);  // raw bits: decoded below
      for (int d = 0; d < W; ++d) {
        if (d == me) continue;
        unsigned long long* w = T.peers[d][2 * me + par].w + 3 + 2 * j;
        ll_store(w, flag, (unsigned)v);
        ll_store(w + 1, flag, (unsigned)(v >> 32));
      }
    }
  }
  // 2. collect this iteration's records from the own mailbox
  if (tid == 0) S.go = 1;
  bool ok = true;
  if (tid < W) {
    unsigned long long k = ~0ULL;
    int i = 0x7FFFFFFF;
    if (tid != me) {
      const unsigned long long* w = T.self_mbox[2 * tid + par].w;
      unsigned lo = 0, hi = 0, ix = 0;
      ok = ll_load(w, flag, lo) && ll_load(w + 1, flag, hi) && ll_load(w + 2, flag, ix);
      k = ((unsigned long long)hi << 32) | lo;
      i = (int)ix;
    }
    S.sh_key[tid] = k;
    S.sh_idx[tid] = i;
  }
  for (int j = tid; j < n_act && ok; j += kThreads) {
    const int a = c.act[j];
    const int s = a % W;
    if (s == me) continue;
    const unsigned long long* w = T.self_mbox[2 * s + par].w + 3 + 2 * j;
    unsigned lo = 0, hi = 0;
    ok = ll_load(w, flag, lo) && ll_load(w + 1, flag, hi);
    rq.prio[a] = __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
  }
  __syncthreads();
  if (!ok) S.go = 0;
  __syncthreads();
  if (!S.go) {
    if (tid == 0) {
      c.status = RS_ECUDA;
      c.error_detail = 10;
    }
    return false;
  }
  // 3. global head: min over shards of (priority bits, rank)
  for (int s = 0; s < W; ++s) {
    const unsigned long long k = S.sh_key[s];
    const int i = S.sh_idx[s];
    if (s != me && (k < key || (k == key && i < idx))) {
      key = k;
      idx = i;
    }
  }
  if (tid == 0) c.alg_bytes += 16LL * n_act + 24LL * W;  // records received
  return true;
}

// The common-configuration kernel's exchange (group G = group M): every shard
// computes the update of every partially prefilled relQuery itself (the update
// is pipelined off the critical path, so replicating it is cheaper than
// exchanging its results), so only the local waiting heads travel: three
// flagged words per shard.  Same mailboxes, flags and parity as shard_exchange.
template <class G>
__device__ bool shard_exchange_heads(const TraceDev& T, Shared& S, unsigned long long& key, int& idx) {
  Ctl& c = S.c;
  const int W = T.shard_world, me = T.shard_rank;
  const int tid = threadIdx.x;
  const unsigned flag = (unsigned)(c.iteration + 1);
  const int par = (int)(c.iteration & 1);
  if (tid < W && tid != me) {
    unsigned long long* w = T.peers[tid][2 * me + par].w;
    ll_store(w + 0, flag, (unsigned)key);
    ll_store(w + 1, flag, (unsigned)(key >> 32));
    ll_store(w + 2, flag, (unsigned)idx);
  }
  if (tid == 0) S.go = 1;
  bool ok = true;
  if (tid < W) {
    unsigned long long k = ~0ULL;
    int i = 0x7FFFFFFF;
    if (tid != me) {
      const unsigned long long* w = T.self_mbox[2 * tid + par].w;
      unsigned lo = 0, hi = 0, ix = 0;
      ok = ll_load(w, flag, lo) && ll_load(w + 1, flag, hi) && ll_load(w + 2, flag, ix);
      k = ((unsigned long long)hi << 32) | lo;
      i = (int)ix;
    }
    S.sh_key[tid] = k;
    S.sh_idx[tid] = i;
  }
  G::sync();
  if (!ok) S.go = 0;
  G::sync();
  if (!S.go) {
    if (tid == 0) {
      c.status = RS_ECUDA;
      c.error_detail = 10;
    }
    return false;
  }
  for (int s = 0; s < W; ++s) {
    const unsigned long long k = S.sh_key[s];
    const int i = S.sh_idx[s];
    if (s != me && (k < key || (k == key && i < idx))) {
      key = k;
      idx = i;
    }
  }
  if (tid == 0) c.alg_bytes += 24LL * W;  // records received
  return true;
}

}  // namespace rsd
