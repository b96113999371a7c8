// pcg64.cuh -- numpy PCG64 (pcg_setseq_128_xsl_rr_64) and
// Generator.choice(n, k, replace=False) replay on the device.
//
// The reference samples its cache-miss ratio with
// `rng.choice(n, size=k, replace=False)` (pkg/src/relsim/prefix_cache.py:157-158)
// on a PCG64 seeded from SeedSequence([seed, 0xD9]) (engine.py:224).  Batch
// decisions depend on the exact sample, so the stream is replayed bit for bit:
// 128-bit LCG step then XSL-RR output, 32-bit half-word buffering, Lemire
// bounded draws, Floyd's algorithm, then the Fisher-Yates pass numpy applies
// to the k results (whose draws must be consumed even though the ratio only
// depends on the sampled set).
#pragma once
#include <stdint.h>

#include "../../include/relserve.h"

namespace rsd {

constexpr uint64_t PCG_MULT_HI = 0x2360ED051FC65DA4ULL;
constexpr uint64_t PCG_MULT_LO = 0x4385DF649FCCF645ULL;

struct Pcg64 {
  uint64_t s_hi, s_lo, i_hi, i_lo;
  uint32_t has32, u32;

  __host__ __device__ static Pcg64 from(const rs_pcg64_state& st) {
    Pcg64 p;
    p.s_hi = st.state_hi;
    p.s_lo = st.state_lo;
    p.i_hi = st.inc_hi;
    p.i_lo = st.inc_lo;
    p.has32 = st.has_uint32;
    p.u32 = st.uinteger;
    return p;
  }
  __host__ __device__ rs_pcg64_state to() const {
    rs_pcg64_state st;
    st.state_hi = s_hi;
    st.state_lo = s_lo;
    st.inc_hi = i_hi;
    st.inc_lo = i_lo;
    st.has_uint32 = has32;
    st.uinteger = u32;
    return st;
  }

  __device__ __forceinline__ uint64_t next64() {
    // state = state * MULT + inc  (mod 2^128)
    const uint64_t lo = s_lo * PCG_MULT_LO;
    uint64_t hi = __umul64hi(s_lo, PCG_MULT_LO) + s_lo * PCG_MULT_HI + s_hi * PCG_MULT_LO;
    const uint64_t nlo = lo + i_lo;
    hi += i_hi + (nlo < lo ? 1ULL : 0ULL);
    s_lo = nlo;
    s_hi = hi;
    const uint64_t x = hi ^ nlo;
    const unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }

  __device__ __forceinline__ uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t v = next64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }

  // random_bounded_uint64(off=0, rng, use_masked=False) for rng < 2^32.
  __device__ __forceinline__ uint32_t bounded(uint32_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return next32();
    const uint32_t excl = rng + 1u;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
      while (left < thr) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

constexpr int kMaxSample = 64;

// Generator.choice(n, k, replace=False) with n < 2^32, k < n, and the Floyd
// branch (not n > 10000 and k > n // 50).  Writes the k sampled indices
// (Floyd order; the shuffle's permutation is applied too).
__device__ __forceinline__ void choice_floyd(Pcg64& g, uint32_t n, uint32_t k, uint32_t* idx) {
  for (uint32_t j = n - k; j < n; ++j) {
    const uint32_t v = g.bounded(j);
    const uint32_t pos = j - (n - k);
    bool found = false;
    for (uint32_t q = 0; q < pos; ++q) found |= (idx[q] == v);
    idx[pos] = found ? j : v;
  }
  for (uint32_t i = k - 1; i >= 1; --i) {
    const uint32_t jj = g.bounded(i);
    const uint32_t t = idx[jj];
    idx[jj] = idx[i];
    idx[i] = t;
  }
}

}  // namespace rsd

namespace rsd {

// ---------------------------------------------------------------------------
// Jump-ahead: s_{t+n} = A^n s_t + C_n (mod 2^128).  tab[i] = (A^(2^i), C_(2^i)).
// Lets every thread start at its own position of the numpy stream, so the
// draws of many Generator.choice calls are produced in parallel and then
// checked for Lemire rejections (which would shift the stream; the caller
// falls back to the sequential replay when one occurs).
// ---------------------------------------------------------------------------
struct U128 {
  uint64_t hi, lo;
};

struct JumpEntry {
  U128 a, c;
};

constexpr int kJumpBits = 32;

__host__ __device__ __forceinline__ U128 mul128(U128 x, U128 y) {
  U128 r;
#ifdef __CUDA_ARCH__
  r.lo = x.lo * y.lo;
  r.hi = __umul64hi(x.lo, y.lo) + x.lo * y.hi + x.hi * y.lo;
#else
  unsigned __int128 p = (unsigned __int128)x.lo * y.lo;
  r.lo = (uint64_t)p;
  r.hi = (uint64_t)(p >> 64) + x.lo * y.hi + x.hi * y.lo;
#endif
  return r;
}

__host__ __device__ __forceinline__ U128 add128(U128 x, U128 y) {
  U128 r;
  r.lo = x.lo + y.lo;
  r.hi = x.hi + y.hi + (r.lo < x.lo ? 1ULL : 0ULL);
  return r;
}

// tab[i] for i < kJumpBits, for a generator with increment inc.
inline void pcg_jump_table(const rs_pcg64_state& st, JumpEntry* tab) {
  U128 a{PCG_MULT_HI, PCG_MULT_LO};
  U128 c{st.inc_hi, st.inc_lo};
  for (int i = 0; i < kJumpBits; ++i) {
    tab[i].a = a;
    tab[i].c = c;
    // (a, c) o (a, c): x -> a(ax + c) + c = a^2 x + (a + 1) c
    U128 one{0, 1};
    c = mul128(add128(a, one), c);
    a = mul128(a, a);
  }
}

// step[k-1] = (A^k, C_k) for k = 1..32.
inline void pcg_step_table(const rs_pcg64_state& st, JumpEntry* step) {
  const U128 A{PCG_MULT_HI, PCG_MULT_LO};
  const U128 inc{st.inc_hi, st.inc_lo};
  U128 a = A, c = inc;
  for (int k = 1; k <= 32; ++k) {
    step[k - 1].a = a;
    step[k - 1].c = c;
    // one more step: x -> A(a x + c) + inc
    c = add128(mul128(A, c), inc);
    a = mul128(A, a);
  }
}

__device__ __forceinline__ U128 pcg_jump(U128 s, unsigned long long n, const JumpEntry* tab) {
  for (int i = 0; n; ++i, n >>= 1)
    if (n & 1ULL) s = add128(mul128(tab[i].a, s), tab[i].c);
  return s;
}

__device__ __forceinline__ uint64_t pcg_output(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

}  // namespace rsd
