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

#include <algorithm>
#include <cmath>
#include <cstring>

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

// ---------------------------------------------------------------------------
// Native reader of the edge-stream CSV format (S/streamio.py:15-79):
//   "# streamtgn-edges v1 d_e=<k>" then "src,dst,t[,f_1..f_k]" per line.
// A fast path only: any line it cannot take as plain decimal fields (or any
// format error) returns STGN_ERR_INVALID with the line number, and the Python
// shim re-reads the file with the reference-faithful parser, so error messages
// and every accepted spelling stay exactly the reference's.
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace {

struct CsvFile {
  std::vector<char> buf;
  bool load(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return false;
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    buf.resize((size_t)(n > 0 ? n : 0) + 1);
    const size_t got = n > 0 ? std::fread(buf.data(), 1, (size_t)n, f) : 0;
    std::fclose(f);
    buf[got] = '\0';
    buf.resize(got + 1);
    return true;
  }
};

const char* skip_ws(const char* p, const char* e) {
  while (p < e && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
  return p;
}

// one field [p, e): strict integer / float, surrounding blanks allowed
bool field_i64(const char* p, const char* e, int64_t* out) {
  p = skip_ws(p, e);
  if (p == e) return false;
  char* end = nullptr;
  errno = 0;
  const long long v = std::strtoll(p, &end, 10);
  if (end == p || errno) return false;
  if (skip_ws(end, e) != e) return false;
  *out = v;
  return true;
}
bool field_f64(const char* p, const char* e, double* out) {
  p = skip_ws(p, e);
  if (p == e) return false;
  for (const char* q = p; q < e; ++q)
    if (*q == 'x' || *q == 'X') return false;  // strtod's hex floats are not Python floats
  char* end = nullptr;
  const double v = std::strtod(p, &end);
  if (end == p) return false;
  if (skip_ws(end, e) != e) return false;
  *out = v;
  return true;
}

// parse everything; on success fills the vectors
int parse_csv(const char* path, int64_t* d_e_out, std::vector<int64_t>& src,
              std::vector<int64_t>& dst, std::vector<double>& t, std::vector<double>& feat,
              int64_t* bad_line) {
  CsvFile f;
  *bad_line = 0;
  if (!f.load(path)) return STGN_ERR_INVALID;
  const char* p = f.buf.data();
  const char* end = p + f.buf.size() - 1;
  static const char kHdr[] = "# streamtgn-edges v1 d_e=";
  const char* nl = p;
  while (nl < end && *nl != '\n') ++nl;
  const size_t hl = sizeof(kHdr) - 1;
  int64_t d_e = 0;
  if ((size_t)(nl - p) < hl || std::strncmp(p, kHdr, hl) != 0 || !field_i64(p + hl, nl, &d_e) ||
      d_e < 0) {
    *bad_line = 1;
    return STGN_ERR_INVALID;
  }
  *d_e_out = d_e;
  int64_t line = 1;
  std::vector<double> row((size_t)d_e);
  p = nl < end ? nl + 1 : end;
  while (p < end) {
    ++line;
    const char* le = p;
    while (le < end && *le != '\n') ++le;
    if (skip_ws(p, le) != le) {
      const char* q = p;
      int64_t s = 0, d = 0;
      double tv = 0.0;
      bool ok = true;
      for (int k = 0; k < 3 + d_e && ok; ++k) {
        const char* fe = q;
        while (fe < le && *fe != ',') ++fe;
        if (k == 0) ok = field_i64(q, fe, &s);
        else if (k == 1) ok = field_i64(q, fe, &d);
        else if (k == 2) ok = field_f64(q, fe, &tv);
        else ok = field_f64(q, fe, &row[(size_t)(k - 3)]);
        if (k < 2 + d_e) {
          if (fe >= le) ok = false;  // too few fields
          q = fe + 1;
        } else {
          if (fe != le) ok = false;  // too many fields
        }
      }
      if (!ok || s < 0 || d < 0) {
        *bad_line = line;
        return STGN_ERR_INVALID;
      }
      src.push_back(s);
      dst.push_back(d);
      t.push_back(tv);
      feat.insert(feat.end(), row.begin(), row.end());
    }
    p = le < end ? le + 1 : end;
  }
  return STGN_OK;
}

}  // namespace

extern "C" int stgn_read_stream(const char* path, int32_t sort, int64_t cap, int64_t* m_out,
                                int64_t* d_e_out, int64_t* src, int64_t* dst, double* t,
                                double* feat, int64_t* bad_line) {
  if (!path || !m_out || !d_e_out || !bad_line) return STGN_ERR_INVALID;
  std::vector<int64_t> s, d;
  std::vector<double> tv, fv;
  const int rc = parse_csv(path, d_e_out, s, d, tv, fv, bad_line);
  if (rc) return rc;
  const int64_t m = (int64_t)s.size(), de = *d_e_out;
  *m_out = m;
  // timestamps must not decrease (S/streamio.py:63-67) unless sort: stable re-sort
  std::vector<int64_t> order((size_t)m);
  for (int64_t i = 0; i < m; ++i) order[(size_t)i] = i;
  // the reference compares each timestamp with the running maximum (NaN never
  // raises it); any NaN is declined so the Python parser decides, and sorting
  // NaN keys would break strict weak ordering
  double run_max = -INFINITY;
  for (int64_t i = 0; i < m; ++i) {
    const double ti = tv[(size_t)i];
    if (std::isnan(ti)) {
      *bad_line = -1;
      return STGN_ERR_INVALID;
    }
    if (ti < run_max && !sort) {
      *bad_line = -1;  // the Python parser reports the exact line
      return STGN_ERR_INVALID;
    }
    run_max = std::max(run_max, ti);
  }
  if (sort) {
    std::stable_sort(order.begin(), order.end(),
                     [&](int64_t a, int64_t b) { return tv[(size_t)a] < tv[(size_t)b]; });
  }
  if (cap < m || !src || !dst || !t || (de && !feat)) return m > cap ? STGN_ERR_CAPACITY : STGN_OK;
  for (int64_t i = 0; i < m; ++i) {
    const int64_t o = order[(size_t)i];
    src[i] = s[(size_t)o];
    dst[i] = d[(size_t)o];
    t[i] = tv[(size_t)o];
    for (int64_t k = 0; k < de; ++k) feat[i * de + k] = fv[(size_t)(o * de + k)];
  }
  return STGN_OK;
}
