// Point ingestion on the device: the reference's
// CsvPointReader (include/geojoin/io.hpp:43-68, src/csv.cpp:26-100) over a text
// buffer in HBM.
//
//   csv_count_newlines_kernel   newlines per 16-byte piece        -> scan
//   csv_line_starts_kernel      start offset of every line
//   csv_parse_rows_kernel       one thread per line: the two named fields,
//                               std::from_chars semantics, latlng_valid
//   (scan of the valid flags, then) csv_scatter_kernel   valid points in order
//
// Decimal -> double is exact (correctly rounded, ties to even) for every
// input, like the fast_float algorithm inside std::from_chars: the decimal
// N * 10^-k is divided bit by bit (restoring division of big integers) until
// 53 significant bits and a round bit are known; the remainder is the sticky
// bit.  Numbers with at most 19 significant digits and k <= 27 (every
// coordinate a program would print) run in 128-bit registers; anything longer
// or smaller runs on 32-bit limbs in local memory.
#pragma once

#include <cstdint>

#include "gj_device.cuh"

namespace gj {

constexpr uint32_t kCsvValid = 0, kCsvInvalid = 1, kCsvEmpty = 2;
constexpr int kCsvMaxDigits = 768;  // beyond this, digits only feed the sticky bit (no double is a tie that late)
constexpr int kCsvLimbs = 120;      // 10^1098 * 2^10 < 2^3660

struct CsvParams {
  const char* text;
  uint64_t n_bytes;          // this chunk
  const uint64_t* line_start;  // [n_lines + 1]; line i is [start[i], start[i + 1] - 1)
  uint64_t n_lines;
  uint32_t lat_index, lng_index;
  uint32_t* status;          // [n_lines]
  uint32_t* valid;           // [n_lines] 1 / 0, for the scan
  double2* point;            // [n_lines] (lat, lng)
  unsigned long long* n_skipped;
  unsigned long long* first_bad;  // min line index (within the chunk) of an invalid row
};

// ---- 128-bit registers ------------------------------------------------------
struct U128 {
  uint64_t lo, hi;
};
__device__ __forceinline__ bool geq(const U128& a, const U128& b) { return a.hi != b.hi ? a.hi > b.hi : a.lo >= b.lo; }
__device__ __forceinline__ void sub(U128& a, const U128& b) {
  const uint64_t borrow = a.lo < b.lo;
  a.lo -= b.lo;
  a.hi -= b.hi + borrow;
}
__device__ __forceinline__ void shl1(U128& a) {
  a.hi = (a.hi << 1) | (a.lo >> 63);
  a.lo <<= 1;
}
__device__ __forceinline__ bool is_zero(const U128& a) { return (a.lo | a.hi) == 0; }

// ---- 32-bit limbs in local memory -------------------------------------------
struct Limbs {
  uint32_t w[kCsvLimbs];
  int n;  // limbs in use (the rest are zero)
};
__device__ inline bool geq(const Limbs& a, const Limbs& b) {
  for (int i = max(a.n, b.n) - 1; i >= 0; --i) {
    if (a.w[i] != b.w[i]) return a.w[i] > b.w[i];
  }
  return true;
}
__device__ inline void sub(Limbs& a, const Limbs& b) {  // a >= b
  uint32_t borrow = 0;
  for (int i = 0; i < a.n; ++i) {
    const uint64_t d = static_cast<uint64_t>(a.w[i]) - b.w[i] - borrow;
    a.w[i] = static_cast<uint32_t>(d);
    borrow = static_cast<uint32_t>(d >> 63);
  }
}
__device__ inline void shl1(Limbs& a) {
  uint32_t carry = 0;
  for (int i = 0; i < a.n; ++i) {
    const uint32_t next = a.w[i] >> 31;
    a.w[i] = (a.w[i] << 1) | carry;
    carry = next;
  }
  if (carry && a.n < kCsvLimbs) a.w[a.n++] = carry;
}
__device__ inline bool is_zero(const Limbs& a) {
  for (int i = 0; i < a.n; ++i) {
    if (a.w[i]) return false;
  }
  return true;
}
__device__ inline void mul_small_add(Limbs& a, uint32_t m, uint32_t add) {
  uint64_t carry = add;
  for (int i = 0; i < a.n; ++i) {
    const uint64_t v = static_cast<uint64_t>(a.w[i]) * m + carry;
    a.w[i] = static_cast<uint32_t>(v);
    carry = v >> 32;
  }
  if (carry && a.n < kCsvLimbs) a.w[a.n++] = static_cast<uint32_t>(carry);
}

// The correctly rounded double of num / (den / 2^10), num < den (i.e. a value
// below 1024), as its bit pattern without the sign; 0 when the value rounds
// to zero.  `sticky`: num stands for something slightly larger (digits that
// were cut off).  Bit t (1-based) of the quotient has weight 2^(10 - t).
template <typename Big>
__device__ inline uint64_t divide_to_double(Big& num, const Big& den, bool sticky) {
  uint64_t z = 0;       // the significant bits so far, leading one included
  int n_sig = 0;        // how many
  int first = 0;        // iteration of the leading one
  // the last bit that can matter is the round bit of the smallest subnormal, 2^-1075
  for (int t = 1; t <= 10 + 1075; ++t) {
    shl1(num);
    uint32_t bit = 0;
    if (geq(num, den)) {
      sub(num, den);
      bit = 1;
    }
    if (n_sig == 0) {
      if (!bit) continue;
      first = t;
    }
    z = (z << 1) | bit;
    if (++n_sig == 54) break;  // 53 + the round bit
  }
  if (n_sig == 0) return 0;  // below 2^-1075
  const bool rest = sticky || !is_zero(num);
  const int e = 10 - first;  // value = 1.xxx * 2^e
  const uint64_t round = z & 1u;
  z >>= 1;
  uint64_t bits;
  if (n_sig == 54 && e >= -1022) {
    bits = (static_cast<uint64_t>(e + 1022) << 52) + z;  // z carries the implicit one into the exponent field
  } else {
    // subnormal: the loop stopped at 2^-1075 (or at 54 bits below the normal range, which the shift fixes)
    int have = n_sig - 1;                 // bits in z
    const int lowest = e - (have - 1);    // weight of z's last bit
    uint64_t r = round;
    bool more = rest;
    for (int w = lowest; w < -1074; ++w) {  // drop bits below 2^-1074 into round / sticky
      more = more || r;
      r = z & 1u;
      z >>= 1;
      --have;
    }
    bits = z + ((r && (more || (z & 1u))) ? 1u : 0u);
    return bits;
  }
  if (round && (rest || (z & 1u))) ++bits;  // ties to even; a carry runs into the exponent by itself
  return bits;
}

__constant__ uint64_t kPow10Lo[28] = {1ull, 10ull, 100ull, 1000ull, 10000ull, 100000ull, 1000000ull, 10000000ull,
                                      100000000ull, 1000000000ull, 10000000000ull, 100000000000ull, 1000000000000ull,
                                      10000000000000ull, 100000000000000ull, 1000000000000000ull, 10000000000000000ull,
                                      100000000000000000ull, 1000000000000000000ull, 10000000000000000000ull,
                                      7766279631452241920ull, 3875820019684212736ull, 1864712049423024128ull,
                                      200376420520689664ull, 2003764205206896640ull, 1590897978359414784ull,
                                      15908979783594147840ull, 11515845246265065472ull};
__constant__ uint64_t kPow10Hi[28] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0,
                                      5ull, 54ull, 542ull, 5421ull, 54210ull, 542101ull, 5421010ull, 54210108ull};

// parse_double (csv.cpp:39-45) + what the caller does with the value: true and
// *out = the double when [b, e) is, after leading blanks, exactly one decimal
// number in std::from_chars' general format whose correctly rounded value is
// finite and not a nonzero decimal rounded to zero.  The words inf / nan parse
// in the reference too, but never give a valid coordinate, so they are
// rejected with everything else.  Values of 1024 and above are rejected
// without being rounded (no coordinate is valid there).
__device__ inline bool csv_parse_double(const char* b, const char* e, double* out) {
  while (b != e && (*b == ' ' || *b == '\t')) ++b;
  const char* p = b;
  bool negative = false;
  if (p != e && *p == '-') {
    negative = true;
    ++p;
  }
  const char* digits_begin = p;
  uint64_t w = 0;          // the first 19 significant digits
  int n_sig = 0;           // significant digits seen (leading zeros excluded)
  int n_digits = 0;        // all digits
  long long q = 0;         // value = w * 10^q (before the explicit exponent)
  bool sticky = false;     // a nonzero digit beyond the 19th
  bool in_fraction = false;
  for (; p != e; ++p) {
    const char c = *p;
    if (c == '.' && !in_fraction) {
      in_fraction = true;
      continue;
    }
    if (c < '0' || c > '9') break;
    ++n_digits;
    const uint32_t d = static_cast<uint32_t>(c - '0');
    if (n_sig == 0 && d == 0) {
      if (in_fraction) --q;
      continue;
    }
    if (n_sig < 19) {
      w = w * 10 + d;
      if (in_fraction) --q;
    } else {
      sticky = sticky || d != 0;
      if (!in_fraction) ++q;
    }
    ++n_sig;
  }
  if (n_digits == 0) return false;
  const char* digits_end = p;
  long long explicit_exp = 0;
  if (p != e && (*p == 'e' || *p == 'E')) {  // a malformed exponent is not consumed
    const char* x = p + 1;
    bool neg = false;
    if (x != e && (*x == '+' || *x == '-')) {
      neg = *x == '-';
      ++x;
    }
    if (x != e && *x >= '0' && *x <= '9') {
      long long ex = 0;
      for (; x != e && *x >= '0' && *x <= '9'; ++x) ex = min(ex * 10 + (*x - '0'), 1000000ll);
      explicit_exp = neg ? -ex : ex;
      q += explicit_exp;
      p = x;
    }
  }
  if (p != e) return false;  // ptr == end (csv.cpp:44)
  const uint64_t sign = negative ? 0x8000000000000000ull : 0ull;
  if (n_sig == 0) {  // all digits zero
    *out = __longlong_as_double(static_cast<long long>(sign));
    return true;
  }
  // decimal exponent of the value: in [10^(dexp - 1), 10^dexp)
  const long long dexp = static_cast<long long>(min(n_sig, 19)) + q;
  if (dexp > 4) return false;     // >= 1000: finite or not, never a coordinate
  if (dexp < -330) return false;  // < 1e-330 rounds to zero: std::errc::result_out_of_range
  uint64_t bits;
  if (q >= 0) {  // a small integer (dexp <= 4 with q >= 0 means at most 4 digits in all)
    uint64_t v = w;
    for (long long k = 0; k < q; ++k) v *= 10;
    *out = __longlong_as_double(static_cast<long long>(sign | static_cast<uint64_t>(__double_as_longlong(static_cast<double>(v)))));
    return true;
  }
  const long long k = -q;
  if (n_sig <= 19 && k <= 27) {  // registers
    U128 num{w, 0};
    U128 den{kPow10Lo[k] << 10, (kPow10Hi[k] << 10) | (kPow10Lo[k] >> 54)};
    if (geq(num, den)) return false;  // >= 1024
    bits = divide_to_double(num, den, false);
  } else {  // limbs: every significant digit up to the 768th, the rest only as a sticky bit
    Limbs num, den;
    num.n = 1;
    num.w[0] = 0;
    int taken = 0;
    bool cut = false, frac = false, lead = true;
    long long q2 = 0;  // value = num * 10^(q2 + explicit_exp), like q for the 19-digit scan
    for (const char* c = digits_begin; c != digits_end; ++c) {
      if (*c == '.') {
        frac = true;
        continue;
      }
      const uint32_t d = static_cast<uint32_t>(*c - '0');
      if (lead && d == 0) {
        if (frac) --q2;
        continue;
      }
      lead = false;
      if (taken < kCsvMaxDigits) {
        mul_small_add(num, 10, d);
        ++taken;
        if (frac) --q2;
      } else {
        cut = cut || d != 0;
        if (!frac) ++q2;
      }
    }
    const long long qq = q2 + explicit_exp;
    if (qq >= 0) return false;    // an integer of 20+ digits: far above any coordinate
    if (-qq > 1098) return false;  // cannot happen with dexp >= -330 and at most 768 digits; defensive
    den.n = 1;
    den.w[0] = 1u << 10;
    for (long long i = 0; i < -qq; ++i) mul_small_add(den, 10, 0);
    for (int i = num.n; i < kCsvLimbs; ++i) num.w[i] = 0;
    for (int i = den.n; i < kCsvLimbs; ++i) den.w[i] = 0;
    num.n = den.n = max(num.n, den.n);
    if (geq(num, den)) return false;  // >= 1024
    bits = divide_to_double(num, den, cut);
  }
  if (bits == 0) return false;                        // a nonzero decimal rounded to zero: range error
  if ((bits >> 52) >= 0x7FFu) return false;           // unreachable below 1024; defensive
  *out = __longlong_as_double(static_cast<long long>(sign | bits));
  return true;
}

// The field_index-th comma-separated field of [b, e) (split_row, csv.cpp:26-37).
__device__ inline bool csv_field(const char* b, const char* e, uint32_t field_index, const char** fb, const char** fe) {
  uint32_t k = 0;
  const char* start = b;
  for (const char* p = b;; ++p) {
    if (p == e || *p == ',') {
      if (k == field_index) {
        *fb = start;
        *fe = p;
        return true;
      }
      if (p == e) return false;
      ++k;
      start = p + 1;
    }
  }
}

// Newlines per 16-byte piece of the text.
__global__ void __launch_bounds__(256)
csv_count_newlines_kernel(const char* __restrict__ text, uint64_t n_bytes, uint32_t* __restrict__ counts) {
  const uint64_t n_pieces = (n_bytes + 15) / 16;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_pieces; i += stride) {
    uint32_t c = 0;
    const uint64_t at = i * 16;
    if (at + 16 <= n_bytes) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(text + at));  // the buffer is 16-byte aligned
      const uint32_t words[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t x = words[k] ^ 0x0A0A0A0Au;  // zero bytes where the newlines are
        c += __popc(((x - 0x01010101u) & ~x & 0x80808080u));
      }
    } else {
      for (uint64_t b = at; b < n_bytes; ++b) c += text[b] == '\n';
    }
    counts[i] = c;
  }
}

// line_start[1 + j] = offset just past the j-th newline.
__global__ void __launch_bounds__(256)
csv_line_starts_kernel(const char* __restrict__ text, uint64_t n_bytes, const uint64_t* __restrict__ offset,
                       uint64_t* __restrict__ line_start) {
  const uint64_t n_pieces = (n_bytes + 15) / 16;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_pieces; i += stride) {
    uint64_t w = offset[i] + 1;
    const uint64_t last = min(n_bytes, i * 16 + 16);
    for (uint64_t b = i * 16; b < last; ++b) {
      if (text[b] == '\n') line_start[w++] = b + 1;
    }
  }
}

// One thread per line (csv.cpp:80-100).
__global__ void __launch_bounds__(128)
csv_parse_rows_kernel(CsvParams cp) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cp.n_lines; i += stride) {
    const char* b = cp.text + cp.line_start[i];
    const char* e = cp.text + cp.line_start[i + 1] - 1;  // without the newline
    if (e != b && e[-1] == '\r') --e;                     // read_line, csv.cpp:47-51
    uint32_t st = kCsvEmpty;
    double lat = 0.0, lng = 0.0;
    if (e != b) {
      const char *ab, *ae, *ob, *oe;
      const bool ok = csv_field(b, e, cp.lat_index, &ab, &ae) && csv_field(b, e, cp.lng_index, &ob, &oe) &&
                      csv_parse_double(ab, ae, &lat) && csv_parse_double(ob, oe, &lng) && latlng_valid(lat, lng);
      st = ok ? kCsvValid : kCsvInvalid;
      if (!ok) {
        atomicAdd(cp.n_skipped, 1ull);
        atomicMin(cp.first_bad, static_cast<unsigned long long>(i));
      }
    }
    cp.status[i] = st;
    cp.valid[i] = st == kCsvValid ? 1u : 0u;
    cp.point[i] = make_double2(lat, lng);
  }
}

__global__ void __launch_bounds__(256)
csv_scatter_kernel(const uint32_t* __restrict__ valid, const uint64_t* __restrict__ offset,
                   const double2* __restrict__ point, uint64_t n_lines, double2* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_lines; i += stride) {
    if (valid[i]) out[offset[i]] = point[i];
  }
}

}  // namespace gj
