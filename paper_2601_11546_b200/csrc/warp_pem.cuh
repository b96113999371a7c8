// warp_pem.cuh -- one warp evaluates the reference's pem() (priority.py:163-218)
// for one remainder, with no block barrier.
//
// Items stream through the warp 32 at a time.  Per chunk the warp takes
// inclusive scans of utok and remaining; the reference's two flush rules --
// close the segment before item j if `utok_j + accum > cap or d_count + 1 >
// mns`, close the prefill sub-batch if `utok_j > 0 and utok_j + p_utok >
// mnbt` -- become a ballot over the lanes at or after the current position,
// and the first set lane is the next event.  Lane 0 adds the fp64 terms in
// the reference's order (sub-batch flushes as they occur; at a segment flush
// the open sub-batch, then the decode term), each one correctly rounded
// (__dmul_rn/__dadd_rn, no FMA).
//
// Every remainder the engine builds has remaining >= 1 for every item and
// utok == 0 for prefilled items (remainder_items, priority.py:81-98), so
// d_count is the item count of the segment and p_utok and accum advance by
// the same utok.  A prefix of prefilled items whose order cannot matter (they
// all fit in the first segment and carry utok 0) may be passed as a summary
// (count, sum and max of remaining) instead of item by item.
#pragma once
#include <stdint.h>

#include "block.cuh"
#include "pem.cuh"

namespace rsd {

struct PrefixSummary {
  int n;          // items (all prefilled, utok 0), n <= mns
  long long rsum; // sum of remaining
  int rmax;       // max remaining
};

// F::item(t, u, rem, pre) for t in [0, n).  Returns the total on every lane.
template <class F>
__device__ double warp_pem(const F& f, int n, const PrefixSummary& pre_sum, const PemModel& m) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  double total = 0.0;
  // segment state (warp-uniform), seeded with the prefilled prefix
  long long accum = 0, p_utok = 0, dsum = pre_sum.rsum;
  long long seg_count = pre_sum.n;
  bool p_ne = false;
  long long lmax = lane == 0 ? pre_sum.rmax : 0;  // per-lane max remaining of the open segment
  const bool any_items = (n + pre_sum.n) > 0;

  for (int base = 0; base < n; base += 32) {
    const int t = base + lane;
    long long u = 0;
    int rem = 0, pre = 1;
    const bool valid = t < n;
    if (valid) f.item(t, u, rem, pre);
    const long long iu = warp_incl_scan(u);
    const long long ir = warp_incl_scan((long long)rem);
    const unsigned vmask = __ballot_sync(kFull, valid);
    const unsigned unp_mask = __ballot_sync(kFull, valid && !pre);
    int s = 0;        // first lane not yet absorbed
    int seg_lo = 0;   // first lane of the open segment within this chunk
    for (;;) {
      const long long iu_before = s > 0 ? __shfl_sync(kFull, iu, s - 1) : 0;
      const long long ir_before = s > 0 ? __shfl_sync(kFull, ir, s - 1) : 0;
      const long long rel_u = iu - iu_before;  // utok of lanes [s, lane]
      const bool in = valid && lane >= s;
      const bool seg_brk = in && (accum + rel_u > m.cap || seg_count + (lane - s) + 1 > m.mns);
      const bool sub_brk = in && u > 0 && p_utok + rel_u > m.mnbt;
      const unsigned ev = __ballot_sync(kFull, seg_brk || sub_brk);
      const int l = ev ? __ffs(ev) - 1 : 32;  // items [s, l) are absorbed
      const int last = (l < 32 ? l : (31 - __clz(vmask | 1u)) + 1);  // one past the last absorbed lane
      if (last > s) {
        const long long du = __shfl_sync(kFull, iu, last - 1) - iu_before;
        const long long dr = __shfl_sync(kFull, ir, last - 1) - ir_before;
        accum += du;
        p_utok += du;
        dsum += dr;
        seg_count += last - s;
        const unsigned span = (last >= 32 ? kFull : ((1u << last) - 1u)) & ~((1u << s) - 1u);
        p_ne = p_ne || (unp_mask & span) != 0;
      }
      if (l >= 32) break;
      const bool is_seg = (__ballot_sync(kFull, seg_brk) >> l) & 1u;
      const long long u_l = __shfl_sync(kFull, u, l);
      const long long r_l = __shfl_sync(kFull, (long long)rem, l);
      const bool unp_l = (unp_mask >> l) & 1u;
      if (is_seg) {
        // flush_segment (priority.py:187-195): open sub-batch, then decode term
        const long long seg_max_lane = (lane >= seg_lo && lane < l && valid) ? (long long)rem : 0;
        long long mx = warp_max(lmax > seg_max_lane ? lmax : seg_max_lane);
        if (p_ne) total = __dadd_rn(total, lin(m.ap, (double)p_utok, m.bp));
        if (seg_count) total = __dadd_rn(total, __dadd_rn(__dmul_rn(m.ad, (double)dsum), __dmul_rn(m.bd, (double)mx)));
        lmax = 0;
        seg_lo = l;
        accum = u_l;
        p_utok = u_l;
        p_ne = unp_l;
        dsum = r_l;
        seg_count = 1;
      } else {
        // prefill sub-batch flush (priority.py:205-208)
        if (p_ne) total = __dadd_rn(total, lin(m.ap, (double)p_utok, m.bp));
        accum += u_l;
        p_utok = u_l;
        p_ne = unp_l;
        dsum += r_l;
        seg_count += 1;
      }
      s = l + 1;
      if (s >= 32) break;
    }
    // fold this chunk's open-segment items into the per-lane max
    if (valid && lane >= seg_lo) lmax = rem > lmax ? rem : lmax;
  }
  if (any_items) {
    const long long mx = warp_max(lmax);
    if (p_ne) total = __dadd_rn(total, lin(m.ap, (double)p_utok, m.bp));
    if (seg_count) total = __dadd_rn(total, __dadd_rn(__dmul_rn(m.ad, (double)dsum), __dmul_rn(m.bd, (double)mx)));
  }
  (void)lt_mask;
  return total;
}

}  // namespace rsd
