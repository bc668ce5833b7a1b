// exsum_core.h — arithmetic shared by the host C++ library and the sm_100a kernels.
//
// Everything here operates on the 67-chunk small-superaccumulator value
// (chunk i weighs 2^(32 i - 1075), small_accumulator.hpp:27-35) and is written
// once for both sides (EXSUM_HD).  None of it is on the per-term hot path; it
// runs once per sum (device: the last CTA / one lane per segment; host: merge,
// round, mean).
//
//   exsum_canonicalize     — carry propagation to the unique canonical form
//                            (semantics of small_accumulator.cpp:244-303)
//   exsum_round_digits     — nearest-even rounding of a base-2^32 magnitude
//                            times 2^scale (semantics of :87-148, oracle.cpp:36-58)
//   exsum_round_canonical  — SmallAccumulator::round on a canonical vector (:330-348)
//   exsum_resolve_specials — Inf/NaN outcome from first-occurrence indices, equal
//                            to the serial add_inf_nan state machine (:230-242)
#ifndef EXSUM_CORE_H_
#define EXSUM_CORE_H_

#include <stdint.h>

#if defined(__CUDACC__)
#define EXSUM_HD __host__ __device__ __forceinline__
#else
#define EXSUM_HD inline
#endif

namespace exsum_b200 {

constexpr int kChunks = 67;               // kSmallChunks
constexpr int kCarryTerms = 2047;         // kSmallCarryTerms
constexpr int kMantBits = 52;
constexpr uint64_t kMantMask = (uint64_t{1} << kMantBits) - 1;
constexpr uint64_t kSignMask = uint64_t{1} << 63;
constexpr uint64_t kPosInf = 0x7FF0000000000000ull;
constexpr uint64_t kNegInf = 0xFFF0000000000000ull;
constexpr uint64_t kCanonicalQnan = 0x7FF8000000000000ull;  // small_accumulator.cpp:29
constexpr uint64_t kNoIndex = ~uint64_t{0};
constexpr int kDigits = kChunks + 1;      // magnitude digits incl. a borrow digit

EXSUM_HD int exsum_clz32(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return __clz(static_cast<int>(x));
#else
  return x ? __builtin_clz(x) : 32;
#endif
}

// Carry propagation.  On return chunks below the top are in [0, 2^32), the top
// chunk is in [-2^32, 2^32), nonzero, and never -1 unless it is chunk 0; every
// chunk above the top is 0.  That representation is unique for a given value,
// so it equals the reference's post-carry_propagate() state whatever sequence
// of adds produced the input.  Returns the top index, or -1 for exact zero.
// Precondition (the reference's add budget): no chunk within 2^32 of overflow.
EXSUM_HD int exsum_canonicalize(int64_t *c) {
  int64_t carry = 0;
  for (int i = 0; i < kChunks - 1; ++i) {
    const int64_t v = c[i] + carry;
    c[i] = v & 0xFFFFFFFFll;
    carry = v >> 32;  // arithmetic: floor division by 2^32
  }
  c[kChunks - 1] += carry;
  int top = kChunks - 1;
  while (top >= 0 && c[top] == 0) --top;
  if (top < 0) return -1;
  // A top chunk of -1 carries only sign information: fold it downward so the
  // top chunk lands in [-2^32, -2] (value unchanged).
  while (top > 0 && c[top] == -1) {
    c[top] = 0;
    --top;
    c[top] -= int64_t{1} << 32;
  }
  return top;
}

// 64 bits of a little-endian base-2^32 digit vector starting at bit `pos`.
EXSUM_HD uint64_t exsum_bits_at(const uint32_t *d, int nd, int pos) {
  const int w = pos >> 5, off = pos & 31;
  const uint64_t d0 = w < nd ? d[w] : 0u;
  const uint64_t d1 = w + 1 < nd ? d[w + 1] : 0u;
  const uint64_t d2 = w + 2 < nd ? d[w + 2] : 0u;
  const uint64_t lo = d0 | (d1 << 32);
  return off ? (lo >> off) | (d2 << (64 - off)) : lo;
}

// True iff any bit strictly below `pos` is set.
EXSUM_HD bool exsum_any_below(const uint32_t *d, int nd, int pos) {
  const int w = pos >> 5, off = pos & 31;
  for (int i = 0; i < w && i < nd; ++i)
    if (d[i]) return true;
  return off && w < nd && (d[w] & ((1u << off) - 1u)) != 0;
}

// Nearest-even double of (-1)^neg * (A + f) * 2^scale, where A = sum d[i] 2^(32 i)
// is nonzero and f in [0, 1) is nonzero iff `sticky`.  The caller guarantees the
// round position lies at or above bit 1 of A whenever sticky is set (true for
// sums, where sticky is never set, and for the mean, which pre-scales A).
EXSUM_HD uint64_t exsum_round_digits(const uint32_t *d, int nd, bool neg, int scale,
                                     bool sticky) {
  const uint64_t sign = neg ? kSignMask : 0;
  int h = nd - 1;
  while (h >= 0 && d[h] == 0) --h;
  if (h < 0) return sign;  // only reachable for A == 0 (not produced by callers)
  const int msb = 32 * h + 31 - exsum_clz32(d[h]);
  const int xexp = msb + scale;            // unbiased exponent of the leading bit
  const bool normal = xexp >= -1022;
  // Position (in A's bits) of the result's unit in the last place.
  const int ulp_pos = normal ? msb - kMantBits : -1074 - scale;
  uint64_t q;
  bool round_bit = false, rest = sticky;
  if (ulp_pos <= 0) {
    q = exsum_bits_at(d, nd, 0) << (-ulp_pos);  // exact (A < 2^53 here)
  } else {
    const uint64_t w = exsum_bits_at(d, nd, ulp_pos - 1);
    q = w >> 1;
    round_bit = (w & 1u) != 0;
    rest = rest || exsum_any_below(d, nd, ulp_pos - 1);
    // q holds at most 53 significant bits (normal) or fewer (denormal)
    q &= (uint64_t{1} << 53) - 1;
  }
  if (round_bit && (rest || (q & 1u))) ++q;
  if (!normal) return sign | q;  // q <= 2^52: denormal, or exactly the least normal
  int biased = xexp + 1023;
  if (q == (uint64_t{1} << 53)) {
    q >>= 1;
    ++biased;
  }
  if (biased >= 2047) return sign | kPosInf;
  return sign | (static_cast<uint64_t>(biased) << kMantBits) | (q & kMantMask);
}

// Magnitude digits of a canonical chunk vector with top index `top` >= 0.
// Returns true for a negative value.  d must hold kDigits entries.
EXSUM_HD bool exsum_magnitude(const int64_t *c, int top, uint32_t *d) {
  const bool neg = c[top] < 0;
  for (int i = 0; i < kDigits; ++i) d[i] = 0;
  if (!neg) {
    for (int i = 0; i <= top; ++i) d[i] = static_cast<uint32_t>(c[i]);
  } else {
    int64_t carry = 0;  // two's-complement negation, borrow-propagating upward
    for (int i = 0; i <= top; ++i) {
      const int64_t v = carry - c[i];
      d[i] = static_cast<uint32_t>(v);
      carry = v >> 32;
    }
    d[top + 1] = static_cast<uint32_t>(carry);
  }
  return neg;
}

// SmallAccumulator::round for a canonical vector (no specials): exact zero is +0.0.
EXSUM_HD uint64_t exsum_round_canonical(const int64_t *c, int top) {
  if (top < 0) return 0;
  uint32_t d[kDigits];
  const bool neg = exsum_magnitude(c, top, d);
  return exsum_round_digits(d, kDigits, neg, -1075, false);
}

// Inf/NaN state of the serial add order given the first index of +Inf (P),
// -Inf (M) and NaN (N) and the NaN's bit pattern.  The serial state machine
// sets nan_bits at the first of {first NaN, first moment both infinities have
// been seen} and inf_bits to the first infinity.
EXSUM_HD void exsum_resolve_specials(uint64_t P, uint64_t M, uint64_t N, uint64_t payload,
                                     uint64_t *inf_bits, uint64_t *nan_bits) {
  const uint64_t both = (P != kNoIndex && M != kNoIndex) ? (P > M ? P : M) : kNoIndex;
  uint64_t nb = 0;
  if (N != kNoIndex && N < both) {
    nb = payload;
  } else if (both != kNoIndex) {
    nb = kCanonicalQnan;
  }
  uint64_t ib = 0;
  if (P != kNoIndex || M != kNoIndex) ib = (P < M) ? kPosInf : kNegInf;
  *inf_bits = ib;
  *nan_bits = nb;
}

EXSUM_HD uint64_t exsum_result_bits(uint64_t inf_bits, uint64_t nan_bits, const int64_t *c,
                                    int top) {
  if (nan_bits) return nan_bits;  // NaN takes precedence (small_accumulator.cpp:331-336)
  if (inf_bits) return inf_bits;
  return exsum_round_canonical(c, top);
}

}  // namespace exsum_b200

#endif  // EXSUM_CORE_H_
