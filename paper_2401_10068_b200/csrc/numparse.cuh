// numparse.cuh -- decimal text -> binary64, correctly rounded, for the dataset loader.
//
// Accepts exactly the syntax Python's float() (and numpy's string -> float64) accepts for
// ASCII input, which is what the reference's reader applies to every CSV field
// (reference cli.py:71-72: float(row[0]), np.array(row[1:], dtype=float)):
//   [ws] [+|-] ( digits [. [digits]] | . digits ) [(e|E) [+|-] digits] [ws]
//   [ws] [+|-] ( inf | infinity | nan ) [ws]            (case-insensitive)
// with single underscores allowed between two digits; ws = str.strip()'s ASCII set.
//
// Conversion: up to 19 significant digits go into a uint64 w with a decimal exponent q;
// Clinger's exact fast path when w < 2^53 and |q| <= 22, otherwise the Eisel-Lemire
// 128-bit product against a table of 5^q (tools/gen_pow5.py), whose result is exact for
// every 19-digit w (Mushtak & Lemire, "Fast number parsing without fallback").  With
// more than 19 significant digits the answer is accepted when EL(w) == EL(w+1) (the
// truncated tail cannot change the rounding); otherwise the field is reported as
// kParseSlow and the caller converts it with the C library's strtod.
//
// The same code is compiled for the host (test hook cv_parse_number_host) and the device.
#pragma once

#include <stdint.h>

namespace cavi {
namespace num {

enum : int { kParseOk = 0, kParseBad = 1, kParseSlow = 2 };

#ifdef __CUDACC__
#define NUM_HD __host__ __device__ __forceinline__
#else
#define NUM_HD inline
#endif

constexpr int kPow5Lo = -342, kPow5Hi = 308;

#ifdef __CUDACC__
__device__ const uint64_t kPow5Dev[] = {
#include "pow5_table.inc"
};
#endif
static const uint64_t kPow5Host[] = {
#include "pow5_table.inc"
};

NUM_HD uint64_t pow5_word(int i) {
#ifdef __CUDA_ARCH__
  return __ldg(kPow5Dev + i);
#else
  return kPow5Host[i];
#endif
}

NUM_HD void mul64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
#ifdef __CUDA_ARCH__
  *lo = a * b;
  *hi = __umul64hi(a, b);
#else
  const unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
#endif
}

NUM_HD int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __clzll((long long)x);
#else
  return __builtin_clzll(x);
#endif
}

NUM_HD double bits_to_double(uint64_t b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  union {
    uint64_t u;
    double d;
  } v;
  v.u = b;
  return v.d;
#endif
}

// Eisel-Lemire: w != 0, q in [kPow5Lo, kPow5Hi]; returns the IEEE bits without sign.
NUM_HD uint64_t eisel_lemire(uint64_t w, int q) {
  const int lz = clz64(w);
  w <<= lz;
  const int idx = 2 * (q - kPow5Lo);
  uint64_t hi, lo;
  mul64(w, pow5_word(idx), &hi, &lo);
  if ((hi & 0x1FFull) == 0x1FFull) {  // the low product can carry into the 55 kept bits
    uint64_t h2, l2;
    mul64(w, pow5_word(idx + 1), &h2, &l2);
    lo += h2;
    if (h2 > lo) ++hi;
  }
  const int upper = (int)(hi >> 63);
  const int shift = upper + 9;
  uint64_t m = hi >> shift;
  // binary exponent: floor(q * log2(10)) + 63 via the 217706 / 2^16 approximation
  int p2 = (((152170 + 65536) * q) >> 16) + 63 + upper - lz + 1023;
  if (p2 <= 0) {  // subnormal or zero
    if (-p2 + 1 >= 64) return 0;
    m >>= -p2 + 1;
    m += m & 1;
    m >>= 1;
    p2 = m < (1ull << 52) ? 0 : 1;
    return (uint64_t)p2 << 52 | (m & ((1ull << 52) - 1));
  }
  // exact halfway between two doubles (possible only for small |q|): round to even
  if (lo <= 1 && q >= -4 && q <= 23 && (m & 3) == 1 && (m << shift) == hi) m &= ~1ull;
  m += m & 1;
  m >>= 1;
  if (m >= (2ull << 52)) {
    m = 1ull << 52;
    ++p2;
  }
  if (p2 >= 0x7FF) return 0x7FFull << 52;
  return (uint64_t)p2 << 52 | (m & ((1ull << 52) - 1));
}

// str.strip()'s ASCII whitespace: space, \t \n \v \f \r and the separators \x1c-\x1f
NUM_HD bool is_ws(char c) { return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f); }
NUM_HD bool is_digit(char c) { return c >= '0' && c <= '9'; }
NUM_HD char lower(char c) { return (c >= 'A' && c <= 'Z') ? (char)(c + 32) : c; }

// case-insensitive match of [p, e) against word
NUM_HD bool match_word(const char* p, const char* e, const char* word) {
  for (; *word; ++word, ++p)
    if (p >= e || lower(*p) != *word) return false;
  return p == e;
}

// Parse [s, e).  On kParseOk *out holds the correctly rounded value.
NUM_HD int parse_double(const char* s, const char* e, double* out) {
  while (s < e && is_ws(*s)) ++s;
  while (e > s && is_ws(e[-1])) --e;
  if (s == e) return kParseBad;
  bool neg = false;
  if (*s == '+' || *s == '-') {
    neg = *s == '-';
    ++s;
  }
  const uint64_t sign = neg ? (1ull << 63) : 0;
  if (s < e && !is_digit(*s) && *s != '.') {
    if (match_word(s, e, "inf") || match_word(s, e, "infinity")) {
      *out = bits_to_double(sign | (0x7FFull << 52));
      return kParseOk;
    }
    if (match_word(s, e, "nan")) {
      *out = bits_to_double(sign | (0x7FFull << 52) | (1ull << 51));
      return kParseOk;
    }
    return kParseBad;
  }
  uint64_t w = 0;
  int nsig = 0;          // significant digits kept in w (<= 19)
  int dropped = 0;       // significant digits beyond 19 (before the point: scale q up)
  bool tail_nonzero = false;
  int frac_kept = 0;     // kept digits after the point
  int ndigits = 0;
  bool seen_point = false;
  char prev = 0;
  for (; s < e; ++s) {
    const char c = *s;
    if (is_digit(c)) {
      ++ndigits;
      const int v = c - '0';
      if (nsig == 0 && v == 0) {
        if (seen_point) ++frac_kept;  // leading zeros after the point still scale
      } else if (nsig < 19) {
        w = w * 10 + (uint64_t)v;
        ++nsig;
        if (seen_point) ++frac_kept;
      } else {
        if (!seen_point) ++dropped;
        tail_nonzero |= v != 0;
      }
    } else if (c == '_') {
      if (!is_digit(prev) || s + 1 >= e || !is_digit(s[1])) return kParseBad;
    } else if (c == '.' && !seen_point) {
      seen_point = true;
    } else {
      break;
    }
    prev = c;
  }
  if (ndigits == 0) return kParseBad;
  int64_t ex = 0;
  if (s < e) {
    if (*s != 'e' && *s != 'E') return kParseBad;
    ++s;
    bool eneg = false;
    if (s < e && (*s == '+' || *s == '-')) {
      eneg = *s == '-';
      ++s;
    }
    int nd = 0;
    prev = 0;
    for (; s < e; ++s) {
      const char c = *s;
      if (is_digit(c)) {
        if (ex < 100000000) ex = ex * 10 + (c - '0');
        ++nd;
      } else if (c == '_') {
        if (!is_digit(prev) || s + 1 >= e || !is_digit(s[1])) return kParseBad;
      } else {
        return kParseBad;
      }
      prev = c;
    }
    if (nd == 0) return kParseBad;
    if (eneg) ex = -ex;
  }
  if (w == 0) {
    *out = bits_to_double(sign);
    return kParseOk;
  }
  const int64_t q64 = ex - frac_kept + dropped;
  if (q64 < kPow5Lo - 19) {  // below half the smallest subnormal even with a 19-digit w
    *out = bits_to_double(sign);
    return kParseOk;
  }
  if (q64 > kPow5Hi) {
    *out = bits_to_double(sign | (0x7FFull << 52));
    return kParseOk;
  }
  int q = (int)q64;
  if (!tail_nonzero && q >= -22 && q <= 22 && w <= (1ull << 53)) {  // Clinger: one exact rounding
    // exact powers of ten 1e0..1e22
    double p = 1.0;
    const int aq = q < 0 ? -q : q;
    double b = 10.0;
    for (int k = aq; k; k >>= 1, b *= b)
      if (k & 1) p *= b;
    const double v = q < 0 ? (double)w / p : (double)w * p;
    *out = neg ? -v : v;
    return kParseOk;
  }
  if (q < kPow5Lo) {
    *out = bits_to_double(sign);
    return kParseOk;
  }
  const uint64_t bits = eisel_lemire(w, q);
  if (tail_nonzero && eisel_lemire(w + 1, q) != bits) return kParseSlow;
  *out = bits_to_double(sign | bits);
  return kParseOk;
}

}  // namespace num
}  // namespace cavi
