// Native synthetic stream generator: the reference's generate_stream
// (S/streamio.py:86-145) for edge-feature-free streams (d_e = 0, the C3/C4
// shapes), producing the identical edge sequence at C speed.
//
// The reference draws from numpy's default_rng(seed) = PCG64 (XSL-RR 128/64).
// The Python shim seeds numpy itself and hands over the resulting bit
// generator state (state, inc, has_uint32, uinteger), so SeedSequence is
// never re-implemented here. The draws reproduced are exactly numpy's:
//   integers(0, k)  -> random_bounded_uint64_fill, k-1 <= 0xFFFFFFFF:
//                      32-bit Lemire with rejection on next_uint32
//                      (0xFFFFFFFF range: plain next_uint32; k-1 = 0: no draw)
//                      k-1 > 0xFFFFFFFF: 64-bit Lemire on next_uint64
//   random()        -> (next_uint64 >> 11) * 2^-53
//   next_uint32     -> half of a 64-bit output, low half first, buffered in
//                      the bit generator (has_uint32 / uinteger)
// standard_normal (the edge features) is not reproduced: streams with d_e > 0
// stay on the Python generator (paper_2603_21090_b200/streamio.py).
#include <stdint.h>
#include <string.h>

#include "stgn.h"

namespace {

typedef unsigned __int128 u128;

struct Pcg64 {
  u128 state, inc;
  int has32;
  uint32_t u32;

  uint64_t next64() {
    const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
    state = state * mult + inc;
    const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t v = next64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)(v & 0xffffffffu);
  }
  double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }

  // numpy Generator.integers(0, k) for int64, k >= 1
  int64_t integers(int64_t k) {
    const uint64_t rng = (uint64_t)(k - 1);
    if (rng == 0) return 0;
    if (rng <= 0xFFFFFFFFull) {
      if (rng == 0xFFFFFFFFull) return (int64_t)next32();
      const uint32_t rng_excl = (uint32_t)rng + 1u;
      uint64_t m = (uint64_t)next32() * rng_excl;
      uint32_t left = (uint32_t)m;
      if (left < rng_excl) {
        const uint32_t thr = (uint32_t)((0xFFFFFFFFu - (uint32_t)rng) % rng_excl);
        while (left < thr) {
          m = (uint64_t)next32() * rng_excl;
          left = (uint32_t)m;
        }
      }
      return (int64_t)(m >> 32);
    }
    if (rng == 0xFFFFFFFFFFFFFFFFull) return (int64_t)next64();
    const uint64_t rng_excl = rng + 1;
    u128 m = (u128)next64() * rng_excl;
    uint64_t left = (uint64_t)m;
    if (left < rng_excl) {
      const uint64_t thr = (0xFFFFFFFFFFFFFFFFull - rng) % rng_excl;
      while (left < thr) {
        m = (u128)next64() * rng_excl;
        left = (uint64_t)m;
      }
    }
    return (int64_t)(uint64_t)(m >> 64);
  }
};

}  // namespace

extern "C" int stgn_generate_stream(const uint64_t* rng_state, int64_t n, int64_t m,
                                    int32_t preferential, double burstiness, int64_t* src,
                                    int64_t* dst, double* t, uint64_t* rng_state_out) {
  if (!rng_state || !src || !dst || !t || n < 2 || m < 1 || !(burstiness >= 1.0))
    return STGN_ERR_INVALID;
  Pcg64 g;
  g.state = ((u128)rng_state[0] << 64) | rng_state[1];
  g.inc = ((u128)rng_state[2] << 64) | rng_state[3];
  g.has32 = rng_state[4] ? 1 : 0;
  g.u32 = (uint32_t)rng_state[5];
  // S/streamio.py:101-104; constants of S/streamio.py:80-81
  const double rate_hi = 2.0 * burstiness / (burstiness + 1.0) * 2.0;
  const double rate_lo = 2.0 / (burstiness + 1.0) * 2.0;
  int64_t hot = (int64_t)((double)n * 0.1);
  if (hot < 2) hot = 2;
  const bool bursty = burstiness > 1.0;
  int64_t k = 0, tick = 0;
  double carry = 0.0;
  // the endpoint pool of the reference is [src_0, dst_0, src_1, dst_1, ...]:
  // pool[j] = j even ? src[j/2] : dst[j/2], so it needs no storage of its own
  while (k < m) {
    const bool is_hot = (tick / 50) % 2 == 1;
    carry += is_hot ? rate_hi : rate_lo;
    const int64_t count = (int64_t)carry;
    carry -= (double)count;
    const int64_t span = (is_hot && bursty) ? hot : n;
    for (int64_t c = 0; c < count && k < m; ++c) {
      const int64_t s = g.integers(span);
      int64_t d;
      if (preferential && k > 0 && g.next_double() < 0.8) {
        const int64_t j = g.integers(2 * k);
        d = (j & 1) ? dst[j >> 1] : src[j >> 1];
      } else {
        d = g.integers(span);
      }
      for (int retry = 0; d == s && retry < 8; ++retry) d = g.integers(span);
      src[k] = s;
      dst[k] = d;
      t[k] = (double)tick;
      ++k;
    }
    ++tick;
  }
  if (rng_state_out) {
    rng_state_out[0] = (uint64_t)(g.state >> 64);
    rng_state_out[1] = (uint64_t)g.state;
    rng_state_out[2] = (uint64_t)(g.inc >> 64);
    rng_state_out[3] = (uint64_t)g.inc;
    rng_state_out[4] = (uint64_t)g.has32;
    rng_state_out[5] = g.u32;
  }
  return STGN_OK;
}
