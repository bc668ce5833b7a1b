// host_accumulators.cpp — host side of the C ABI: the small and large
// superaccumulator objects and the partial-record helpers.
//
// These are the reference's caller-owned accumulator objects re-expressed in
// C++ behind the C ABI.  They run on the CPU by design, as
// their reference counterparts do (small_accumulator.cpp, large_accumulator.cpp);
// the data-parallel hot path (exact sum of a whole array) is the device path in
// sum_kernels.cu and never falls back to this file.
//
// Arithmetic follows the paper (Neal 2015, Fig. 3 and Fig. 4):
//   small add      — two signed 64-bit chunk updates per term, carry budget 2047
//   large add      — raw-bits accumulation per sign+exponent index with a 4096
//                    countdown, transfer as three 32-bit pieces into the small one
// Canonicalisation, rounding and the mean share exsum_core.h with the kernels.

#include <cstdint>
#include <cstring>
#include <new>

#if defined(__x86_64__) && !defined(EXSUM_NO_AVX512)
#include <immintrin.h>
#define EXSUM_HAVE_AVX512 1
#else
#define EXSUM_HAVE_AVX512 0
#endif

#include "exsum_b200.h"
#include "exsum_core.h"

using namespace exsum_b200;

#ifndef EXSUM_SMALL_COPIES
#define EXSUM_SMALL_COPIES 2  // local chunk arrays taken in turn by add(span) (store-forwarding chains)
#endif

namespace {

inline uint64_t bits_of(double v) {
  uint64_t b;
  std::memcpy(&b, &v, sizeof b);
  return b;
}

inline double double_of(uint64_t b) {
  double v;
  std::memcpy(&v, &b, sizeof v);
  return v;
}

// ------------------------------------------------------------ small accumulator

// add_inf_nan semantics (small_accumulator.cpp:230-242): the first NaN keeps its
// payload; a second, different infinity turns the result into the canonical NaN.
inline void small_special(exsum_small *a, uint64_t bits) {
  if ((bits & kMantMask) == 0) {
    if (a->inf_bits == 0) {
      a->inf_bits = bits;
    } else if (a->inf_bits != bits && a->nan_bits == 0) {
      a->nan_bits = kCanonicalQnan;
    }
  } else if (a->nan_bits == 0) {
    a->nan_bits = bits;
  }
}

// Fig. 3: split the 53-bit significand, positioned by the low five exponent
// bits, into a low 32-bit piece for chunk e>>5 and the rest for the next chunk.
// Returns false for terms that leave the chunks untouched (+-0, Inf, NaN).
inline bool small_add_term(exsum_small *a, uint64_t bits) {
  const uint32_t e = static_cast<uint32_t>(bits >> kMantBits) & 0x7FFu;
  uint64_t m = bits & kMantMask;
  uint32_t ee = e;
  if (e == 0x7FFu) {
    small_special(a, bits);
    return false;
  }
  if (e == 0) {
    if (m == 0) return false;
    ee = 1;  // denormal: exponent 1 without the implicit bit
  } else {
    m |= uint64_t{1} << kMantBits;
  }
  const uint32_t sh = ee & 31u;
  const uint32_t ix = ee >> 5;
  const int64_t low = static_cast<int64_t>((m << sh) & 0xFFFFFFFFull);
  const int64_t high = static_cast<int64_t>(m >> (32u - sh));
  if (bits >> 63) {
    a->chunk[ix] -= low;
    a->chunk[ix + 1] -= high;
  } else {
    a->chunk[ix] += low;
    a->chunk[ix + 1] += high;
  }
  return true;
}

inline int small_propagate(exsum_small *a) {
  a->adds_until_propagate = kCarryTerms;
  return exsum_canonicalize(a->chunk);
}

void small_zero(exsum_small *a) {
  std::memset(a, 0, sizeof *a);
  a->adds_until_propagate = kCarryTerms;
}

// Magnitude, sign and top of an accumulator after propagation.
struct Mag {
  uint32_t d[kDigits + 4];
  int nd;
  bool neg;
};

// Correctly rounded (value / n), value = A * 2^-1075.  The quotient is formed
// with enough extra low bits that the rounding position is at least two bits
// above the division's truncation point, the remainder feeding the sticky bit.
uint64_t mean_bits(const int64_t *c, int top, uint64_t n) {
  uint32_t d[kDigits];
  const bool neg = exsum_magnitude(c, top, d);
  int h = kDigits - 1;
  while (h > 0 && d[h] == 0) --h;
  const int alen = 32 * h + 32 - exsum_clz32(d[h]);
  int nlen = 64;
  while (nlen > 1 && !((n >> (nlen - 1)) & 1u)) --nlen;
  int t = 55 + nlen - alen + 1;
  if (t < 2) t = 2;
  // num = A << t, as digits (t < 32 * 8 always: alen >= 2, nlen <= 64)
  constexpr int kMax = kDigits + 8;
  uint32_t num[kMax] = {};
  const int ws = t >> 5, bs = t & 31;
  for (int i = 0; i < kDigits; ++i) {
    const uint64_t v = static_cast<uint64_t>(d[i]) << bs;
    num[i + ws] |= static_cast<uint32_t>(v);
    if (i + ws + 1 < kMax) num[i + ws + 1] |= static_cast<uint32_t>(v >> 32);
  }
  // Long division by n (remainder < n < 2^64, so rem:digit fits in 96 bits).
  unsigned __int128 rem = 0;
  for (int i = kMax - 1; i >= 0; --i) {
    const unsigned __int128 cur = (rem << 32) | num[i];
    num[i] = static_cast<uint32_t>(cur / n);
    rem = cur % n;
  }
  return exsum_round_digits(num, kMax, neg, -1075 - t, rem != 0);
}

// ------------------------------------------------------------ large accumulator

constexpr int kBins = 4096;
constexpr int kBinAdds = 4096;  // kLargeChunkAdds: 12 spare bits above the mantissa

}  // namespace

struct exsum_large {
  uint64_t word[kBins];    // wrapped sum of raw bit patterns, valid while in use
  int16_t left[kBins];     // adds remaining before a transfer; -1 = not in use
  uint64_t used[kBins / 64];
  uint64_t used_words;
  exsum_small small;
};

namespace {

// Transfer of one bin into the small accumulator (paper §large; reference
// large_accumulator.cpp:59-111).  The bin holds sum of (4096 - left) raw
// patterns; adding index*left at bit 52 completes the index bits to a multiple
// of 2^64, leaving the mantissa-field sum; the implicit ones (one per add) are
// re-inserted above it; the 96-bit window is applied as three 32-bit pieces.
void large_transfer(exsum_large *L, uint32_t ix) {
  exsum_small *s = &L->small;
  if (s->adds_until_propagate < 3) small_propagate(s);
  const int64_t left = L->left[ix];
  uint64_t w = L->word[ix];
  if (left > 0) w += (static_cast<uint64_t>(left) * ix) << kMantBits;
  const uint32_t e = ix & 0x7FFu;
  const uint32_t sh = e ? (e & 31u) : 1u;
  const uint32_t base = e ? (e >> 5) : 0u;
  const uint64_t p0 = (w << sh) & 0xFFFFFFFFull;
  uint64_t mid = w >> (32u - sh);
  if (e) mid += static_cast<uint64_t>(kBinAdds - left) << (kMantBits - 32 + sh);
  const uint64_t p2 = mid >> 32;
  const uint64_t p1 = mid & 0xFFFFFFFFull;
  const int64_t sgn = (ix >> 11) ? -1 : 1;
  s->chunk[base] += sgn * static_cast<int64_t>(p0);
  s->chunk[base + 1] += sgn * static_cast<int64_t>(p1);
  s->chunk[base + 2] += sgn * static_cast<int64_t>(p2);
  s->adds_until_propagate -= 3;
}

// The rare branch of an add (decremented count negative): Inf/NaN, first use
// of a bin, or a bin that has absorbed its 4096 adds.
void large_slow(exsum_large *L, uint32_t ix, uint64_t bits) {
  if ((ix & 0x7FFu) == 0x7FFu) {  // Inf/NaN: bin stays unused
    small_special(&L->small, bits);
    return;
  }
  if (L->left[ix] >= 0) large_transfer(L, ix);  // full bin (left == 0)
  L->word[ix] = bits;
  L->left[ix] = kBinAdds - 1;
  L->used[ix >> 6] |= uint64_t{1} << (ix & 63u);
  L->used_words |= uint64_t{1} << (ix >> 6);
}

inline void large_add_bits(exsum_large *L, uint64_t bits) {
  const uint32_t ix = static_cast<uint32_t>(bits >> kMantBits);
  const int left = L->left[ix] - 1;
  if (left < 0) {
    large_slow(L, ix, bits);
  } else {
    L->left[ix] = static_cast<int16_t>(left);
    L->word[ix] += bits;
  }
}

void large_reset(exsum_large *L) {
  for (int i = 0; i < kBins; ++i) L->left[i] = -1;
  std::memset(L->used, 0, sizeof L->used);
  L->used_words = 0;
  small_zero(&L->small);
}

void large_drain(exsum_large *L) {
  uint64_t words = L->used_words;
  while (words) {
    const int w = __builtin_ctzll(words);
    uint64_t flags = L->used[w];
    while (flags) {
      const uint32_t ix = static_cast<uint32_t>(w * 64 + __builtin_ctzll(flags));
      if (L->left[ix] >= 0 && L->left[ix] < kBinAdds) large_transfer(L, ix);
      L->left[ix] = -1;
      flags &= flags - 1;
    }
    L->used[w] = 0;
    words &= words - 1;
  }
  L->used_words = 0;
}

}  // namespace

// ================================================================== C ABI

extern "C" {

int exsum_small_init(exsum_small *acc) {
  if (!acc) return EXSUM_EINVAL;
  small_zero(acc);
  return EXSUM_OK;
}

int exsum_small_add(exsum_small *acc, double v) {
  if (!acc) return EXSUM_EINVAL;
  if (acc->adds_until_propagate <= 0) small_propagate(acc);
  if (small_add_term(acc, bits_of(v))) --acc->adds_until_propagate;
  return EXSUM_OK;
}

// add(span) (small_accumulator.cpp:174-189): the same runs between
// propagations, but each run is summed branch-free (sign applied as
// (v ^ s) - s, no mispredicted sign branch on mixed-sign data) into
// EXSUM_SMALL_COPIES local chunk arrays taken in turn (no store-to-load chain
// through the same chunk on consecutive terms), then added to the accumulator.  Integer adds
// are associative and a run stays within the 2047-add budget, so the chunk
// values after every call equal the reference's sequential adds exactly.
// One term of a run (small_add_term's arithmetic) into the local chunk array cj:
// branch-free sign ((v ^ s) - s); zeros skipped, denormals at exponent 1, Inf/NaN
// to the accumulator's special state.
static inline void small_term_local(exsum_small *acc, int64_t *cj, uint64_t bits) {
  const uint32_t e = static_cast<uint32_t>(bits >> kMantBits) & 0x7FFu;
  uint64_t m = bits & kMantMask;
  uint32_t ee = e;
  if (__builtin_expect(e - 1u >= 0x7FEu, 0)) {  // e == 0 or e == 0x7FF
    if (e == 0x7FFu) {
      small_special(acc, bits);
      return;
    }
    if (m == 0) return;
    ee = 1;
  } else {
    m |= uint64_t{1} << kMantBits;
  }
  const uint32_t sh = ee & 31u, ix = ee >> 5;
  const int64_t s = static_cast<int64_t>(bits) >> 63;  // 0 or -1
  const int64_t low = static_cast<int64_t>((m << sh) & 0xFFFFFFFFull);
  const int64_t high = static_cast<int64_t>(m >> (32u - sh));
  cj[ix] += (low ^ s) - s;
  cj[ix + 1] += (high ^ s) - s;
}

// AVX-512 form of a run's adds for the common case: 8 terms at a time whose
// exponent fields are all in [1, 2046] (no zero, denormal, Inf or NaN) and
// share one chunk index e >> 5 (every U[-1,1) term but those below 2^-31, for
// example).  Such groups are split exactly as small_add_term does and summed in
// two vector accumulators (chunk ix and ix + 1; per-lane sums stay below 2^43
// and 2^63 within a run); a group that does not qualify returns to the scalar
// loop at its first term.  Returns how many terms of [0, run) it consumed.
#if EXSUM_HAVE_AVX512
__attribute__((target("avx512f"))) static size_t small_run_avx512(const uint64_t *b, size_t run,
                                                           int64_t *c) {
  const __m512i kMask11 = _mm512_set1_epi64(0x7FF), kMant = _mm512_set1_epi64(kMantMask),
                kOne = _mm512_set1_epi64(int64_t{1} << kMantBits),
                kLow = _mm512_set1_epi64(0xFFFFFFFFll), k32 = _mm512_set1_epi64(32),
                k31 = _mm512_set1_epi64(31), k1 = _mm512_set1_epi64(1),
                kSpan = _mm512_set1_epi64(0x7FE);
  __m512i accl = _mm512_setzero_si512(), acch = _mm512_setzero_si512();
  int64_t hot = -1;
  size_t j = 0;
  for (; j + 8 <= run; j += 8) {
    const __m512i v = _mm512_loadu_si512(b + j);
    const __m512i e = _mm512_and_si512(_mm512_srli_epi64(v, kMantBits), kMask11);
    const __m512i ix = _mm512_srli_epi64(e, 5);
    const __m512i ix0 = _mm512_permutexvar_epi64(_mm512_setzero_si512(), ix);
    // all normal (e - 1 < 2046 unsigned) and one chunk index
    const __mmask8 ok = _mm512_cmplt_epu64_mask(_mm512_sub_epi64(e, k1), kSpan) &
                        _mm512_cmpeq_epi64_mask(ix, ix0);
    if (ok != 0xFF) break;
    const int64_t gix = _mm512_cvtsi512_si32(ix0);
    if (gix != hot) {
      if (hot >= 0) {
        c[hot] += _mm512_reduce_add_epi64(accl);
        c[hot + 1] += _mm512_reduce_add_epi64(acch);
        accl = _mm512_setzero_si512();
        acch = _mm512_setzero_si512();
      }
      hot = gix;
    }
    const __m512i m = _mm512_or_si512(_mm512_and_si512(v, kMant), kOne);
    const __m512i sh = _mm512_and_si512(e, k31);
    const __m512i low = _mm512_and_si512(_mm512_sllv_epi64(m, sh), kLow);
    const __m512i high = _mm512_srlv_epi64(m, _mm512_sub_epi64(k32, sh));
    const __m512i sg = _mm512_srai_epi64(v, 63);  // 0 or -1
    accl = _mm512_add_epi64(accl, _mm512_sub_epi64(_mm512_xor_si512(low, sg), sg));
    acch = _mm512_add_epi64(acch, _mm512_sub_epi64(_mm512_xor_si512(high, sg), sg));
  }
  if (hot >= 0) {
    c[hot] += _mm512_reduce_add_epi64(accl);
    c[hot + 1] += _mm512_reduce_add_epi64(acch);
  }
  return j;
}

static bool have_avx512() {
  static const bool yes = __builtin_cpu_supports("avx512f");
  return yes;
}
#endif

int exsum_small_add_array(exsum_small *acc, const double *x, size_t n) {
  if (!acc || (n && !x)) return EXSUM_EINVAL;
  size_t i = 0;
  while (i < n) {
    if (acc->adds_until_propagate <= 0) small_propagate(acc);
    size_t run = static_cast<size_t>(acc->adds_until_propagate);
    if (run > n - i) run = n - i;
    int64_t c[EXSUM_SMALL_COPIES][kChunks + 1] = {};
    size_t j = 0;
#if EXSUM_HAVE_AVX512
    // vector groups first, then the scalar loop from the first group that did
    // not qualify; the vector path re-enters after every scalar stretch of 8
    while (j < run && have_avx512()) {
      j += small_run_avx512(reinterpret_cast<const uint64_t *>(x + i) + j, run - j, c[0]);
      if (j + 8 > run) break;
      const size_t stop = j + 8;  // one group's worth through the scalar loop
      for (; j < stop; ++j) small_term_local(acc, c[j % EXSUM_SMALL_COPIES], bits_of(x[i + j]));
    }
#endif
    for (; j < run; ++j) small_term_local(acc, c[j % EXSUM_SMALL_COPIES], bits_of(x[i + j]));
    for (int k = 0; k < kChunks; ++k) {
      int64_t t = 0;
      for (int r = 0; r < EXSUM_SMALL_COPIES; ++r) t += c[r][k];
      acc->chunk[k] += t;
    }
    acc->adds_until_propagate -= static_cast<int32_t>(run);  // budget per element
    i += run;
  }
  return EXSUM_OK;
}

int exsum_small_add_inf_nan(exsum_small *acc, uint64_t bits) {
  if (!acc || ((bits >> kMantBits) & 0x7FFu) != 0x7FFu) return EXSUM_EINVAL;
  small_special(acc, bits);
  return EXSUM_OK;
}

int exsum_small_carry_propagate(exsum_small *acc) {
  if (!acc) return -1;
  return small_propagate(acc);
}

int exsum_small_merge(exsum_small *dst, const exsum_small *src) {
  if (!dst || !src) return EXSUM_EINVAL;
  exsum_small s = *src;
  small_propagate(&s);
  if (s.nan_bits && !dst->nan_bits) dst->nan_bits = s.nan_bits;
  if (s.inf_bits) {
    if (!dst->inf_bits) {
      dst->inf_bits = s.inf_bits;
    } else if (dst->inf_bits != s.inf_bits && !dst->nan_bits) {
      dst->nan_bits = kCanonicalQnan;
    }
  }
  for (int i = 0; i < kChunks; ++i) dst->chunk[i] += s.chunk[i];
  small_propagate(dst);
  return EXSUM_OK;
}

int exsum_small_round(exsum_small *acc, double *out) {
  if (!acc || !out) return EXSUM_EINVAL;
  if (acc->nan_bits) {
    *out = double_of(acc->nan_bits);
  } else if (acc->inf_bits) {
    *out = double_of(acc->inf_bits);
  } else {
    const int top = small_propagate(acc);
    *out = double_of(exsum_round_canonical(acc->chunk, top));
  }
  return EXSUM_OK;
}

int exsum_small_mean(exsum_small *acc, uint64_t n, double *out) {
  if (!acc || !out || n == 0) return EXSUM_EINVAL;
  if (acc->nan_bits) {
    *out = double_of(acc->nan_bits);
  } else if (acc->inf_bits) {
    *out = double_of(acc->inf_bits);
  } else {
    const int top = small_propagate(acc);
    *out = top < 0 ? 0.0 : double_of(mean_bits(acc->chunk, top, n));
  }
  return EXSUM_OK;
}

exsum_large *exsum_large_new(void) {
  exsum_large *L = new (std::nothrow) exsum_large;
  if (L) large_reset(L);
  return L;
}

void exsum_large_free(exsum_large *acc) { delete acc; }

int exsum_large_add(exsum_large *acc, double v) {
  if (!acc) return EXSUM_EINVAL;
  large_add_bits(acc, bits_of(v));
  return EXSUM_OK;
}

int exsum_large_add_array(exsum_large *acc, const double *x, size_t n) {
  if (!acc || (n && !x)) return EXSUM_EINVAL;
  for (size_t i = 0; i < n; ++i) large_add_bits(acc, bits_of(x[i]));
  return EXSUM_OK;
}

int exsum_large_drain(exsum_large *acc) {
  if (!acc) return EXSUM_EINVAL;
  large_drain(acc);
  return EXSUM_OK;
}

int exsum_large_round(exsum_large *acc, double *out) {
  if (!acc || !out) return EXSUM_EINVAL;
  large_drain(acc);
  return exsum_small_round(&acc->small, out);
}

int exsum_large_mean(exsum_large *acc, uint64_t n, double *out) {
  if (!acc || !out || n == 0) return EXSUM_EINVAL;
  large_drain(acc);
  return exsum_small_mean(&acc->small, n, out);
}

int exsum_large_small(const exsum_large *acc, exsum_small *out) {
  if (!acc || !out) return EXSUM_EINVAL;
  *out = acc->small;
  return EXSUM_OK;
}

int exsum_large_count(const exsum_large *acc, int ix, int *count) {
  if (!acc || !count || ix < 0 || ix >= kBins) return EXSUM_EINVAL;
  *count = acc->left[ix];
  return EXSUM_OK;
}

int exsum_large_chunk_in_use(const exsum_large *acc, int ix) {
  if (!acc || ix < 0 || ix >= kBins) return 0;
  return static_cast<int>((acc->used[ix >> 6] >> (ix & 63)) & 1u);
}

int exsum_large_chunk_word(const exsum_large *acc, int ix, uint64_t *word) {
  if (!acc || !word || ix < 0 || ix >= kBins) return EXSUM_EINVAL;
  *word = acc->word[ix];
  return EXSUM_OK;
}

int exsum_large_chunks_in_use(const exsum_large *acc) {
  if (!acc) return 0;
  int used = 0;
  for (int i = 0; i < kBins; ++i) used += acc->left[i] >= 0;
  return used;
}

// ---------------------------------------------------------- sqnorm / dot

// sum_products (vector_ops.cpp:72-97) with SumMethod::large: every product is
// rounded by the host multiply (the reference's a[i] * b[i], same x86 rules for
// NaN operands and 0 * Inf), then summed exactly — by the host kernel of
// host_sum.cpp, on every hardware thread for long vectors (exsum_host_products).
// Built without FMA contraction (baseline x86-64), like the reference's products.
int exsum_sqnorm(const double *x, size_t n, double *out) {
  if (!out || (n && !x)) return EXSUM_EINVAL;
  return exsum_host_products(x, x, n, 0, out);
}

int exsum_dot(const double *a, size_t na, const double *b, size_t nb, double *out) {
  if (!out || na != nb || (na && (!a || !b))) return EXSUM_EINVAL;  // vector_ops.cpp:150-152
  return exsum_host_products(a, b, na, 0, out);
}

// ------------------------------------------------------------ partial records

int exsum_partial_from_array(const double *x, size_t n, uint64_t base_index,
                             exsum_partial *out) {
  if (!out || (n && !x)) return EXSUM_EINVAL;
  exsum_large *L = exsum_large_new();
  if (!L) return EXSUM_ENOMEM;
  uint64_t P = kNoIndex, M = kNoIndex, N = kNoIndex, payload = 0;
  for (size_t i = 0; i < n; ++i) {
    const uint64_t b = bits_of(x[i]);
    if (((b >> kMantBits) & 0x7FFu) == 0x7FFu) {
      const uint64_t gi = base_index + i;
      if (b & kMantMask) {
        if (N == kNoIndex) {
          N = gi;
          payload = b;
        }
      } else if (b >> 63) {
        if (M == kNoIndex) M = gi;
      } else if (P == kNoIndex) {
        P = gi;
      }
      continue;
    }
    large_add_bits(L, b);
  }
  large_drain(L);
  out->acc = L->small;
  exsum_large_free(L);
  small_propagate(&out->acc);
  exsum_resolve_specials(P, M, N, payload, &out->acc.inf_bits, &out->acc.nan_bits);
  out->acc.reserved_ = 0;
  out->first_pos_inf = P;
  out->first_neg_inf = M;
  out->first_nan = N;
  out->nan_payload = payload;
  return EXSUM_OK;
}

int exsum_partial_merge(const exsum_partial *parts, size_t k, exsum_partial *out,
                        double *result) {
  if (!parts && k) return EXSUM_EINVAL;
  int64_t c[kChunks] = {};
  uint64_t P = kNoIndex, M = kNoIndex, N = kNoIndex, payload = 0;
  for (size_t j = 0; j < k; ++j) {
    exsum_small s = parts[j].acc;
    exsum_canonicalize(s.chunk);  // each addend within 2^33: no overflow for k < 2^29
    for (int i = 0; i < kChunks; ++i) c[i] += s.chunk[i];
    if (parts[j].first_pos_inf < P) P = parts[j].first_pos_inf;
    if (parts[j].first_neg_inf < M) M = parts[j].first_neg_inf;
    if (parts[j].first_nan < N) {
      N = parts[j].first_nan;
      payload = parts[j].nan_payload;
    }
  }
  const int top = exsum_canonicalize(c);
  uint64_t ib, nb;
  exsum_resolve_specials(P, M, N, payload, &ib, &nb);
  if (result) *result = double_of(exsum_result_bits(ib, nb, c, top));
  if (out) {
    std::memcpy(out->acc.chunk, c, sizeof c);
    out->acc.inf_bits = ib;
    out->acc.nan_bits = nb;
    out->acc.adds_until_propagate = kCarryTerms;
    out->acc.reserved_ = 0;
    out->first_pos_inf = P;
    out->first_neg_inf = M;
    out->first_nan = N;
    out->nan_payload = payload;
  }
  return EXSUM_OK;
}

int exsum_partial_round(const exsum_partial *p, double *out) {
  if (!p || !out) return EXSUM_EINVAL;
  exsum_small s = p->acc;
  return exsum_small_round(&s, out);
}

}  // extern "C"
