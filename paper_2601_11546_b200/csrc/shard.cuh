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
// shards run on one GPU), fences, publishes a sequence number, and spins on the
// sequence numbers of its own mailbox.  Records are double-buffered by
// iteration parity: a shard can only reach iteration t+2 after every shard
// published t+1, which each does only after consuming t's records.
#pragma once
#include "engine_state.cuh"

namespace rsd {

// One shard's record for one iteration.  prios[j] is valid for the act-list
// positions j whose relQuery the sender owns.
struct alignas(16) ShardRec {
  unsigned long long seq;  // iteration + 1 once the record is complete
  unsigned long long key;  // local waiting head: priority bits (~0 if none)
  int idx;                 // local waiting head: admission rank
  int pad;
  unsigned long long pad2;
  double prios[kMaxAct];
};

// A shard's mailbox: ShardRec[world][2] (sender, iteration parity).
__host__ __device__ inline size_t mailbox_bytes(int world) { return sizeof(ShardRec) * 2 * (size_t)world; }

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// All threads.  In: this shard's local head (key, idx), its owned priorities in
// rq.prio.  Out: the global head in (key, idx); every owned-elsewhere priority
// of the act list written into this replica's rq.prio.  Returns false on an
// exchange timeout (status set; every shard then stops).
__device__ bool shard_exchange(const TraceDev& T, Shared& S, unsigned long long& key, int& idx) {
  Ctl& c = S.c;
  const RqView& rq = S.rq;
  const int W = T.shard_world, me = T.shard_rank;
  const int tid = threadIdx.x;
  const unsigned long long seq = (unsigned long long)c.iteration + 1;
  const int par = (int)(c.iteration & 1);
  const int n_act = c.n_act;
  // 1. owned priorities into every peer's mailbox slot [me][par]
  for (int j = tid; j < n_act; j += kThreads) {
    const int a = c.act[j];
    if (a % W == me) {
      const double v = rq.prio[a];
      for (int d = 0; d < W; ++d)
        if (d != me) T.peers[d][2 * me + par].prios[j] = v;
    }
  }
  __threadfence_system();
  __syncthreads();
  // 2. headers, sequence number last (release)
  if (tid < W && tid != me) {
    ShardRec* r = &T.peers[tid][2 * me + par];
    r->key = key;
    r->idx = idx;
    st_release_sys(&r->seq, seq);
  }
  // 3. wait for every other shard's record of this iteration
  if (tid == 0) S.go = 1;
  __syncthreads();
  if (tid < W && tid != me) {
    const unsigned long long* sp = &T.self_mbox[2 * tid + par].seq;
    const long long t0 = clock64();
    while (ld_acquire_sys(sp) != seq) {
      if (clock64() - t0 > (1LL << 33)) {  // ~4 s at 2 GHz: a peer is gone
        S.go = 0;
        break;
      }
    }
  }
  __syncthreads();
  if (!S.go) {
    if (tid == 0) {
      c.status = RS_ECUDA;
      c.error_detail = 10;
    }
    return false;
  }
  // 4. global head and the other shards' priorities (L2 reads: bypass L1)
  for (int s = 0; s < W; ++s) {
    if (s == me) continue;
    const ShardRec* r = &T.self_mbox[2 * s + par];
    const unsigned long long k = __ldcg(&r->key);
    const int i = __ldcg(&r->idx);
    if (k < key || (k == key && i < idx)) {
      key = k;
      idx = i;
    }
  }
  for (int j = tid; j < n_act; j += kThreads) {
    const int a = c.act[j];
    const int s = a % W;
    if (s != me) rq.prio[a] = __ldcg(&T.self_mbox[2 * s + par].prios[j]);
  }
  if (tid == 0) c.alg_bytes += 8LL * n_act + 16LL * W;  // records received
  __syncthreads();
  return true;
}

}  // namespace rsd
