// sum_kernels.cu — the sm_100a exact-summation hot path.
//
// Replaces exact_sum(values, ExactMethod::large) (vector_ops.cpp:121-130), i.e.
// LargeAccumulator::add(span) + drain + SmallAccumulator::round
// (large_accumulator.cpp:28-136, small_accumulator.cpp:244-348), and the
// split-merge of parallel_exact_sum (vector_ops.cpp:172-186).  See DESIGN.md.
//
// Device representation (B200-first, not the reference's): every LANE owns a
// private fixed-point superaccumulator in shared memory, so a term costs one
// conflict-free shared read-modify-write and a handful of integer instructions
// — no atomics, no bank conflicts, no dependence on how exponents are
// distributed.  Two slot layouts are built (EXSUM_SLOT_BITS):
//
//   128 (default)  slot k = signed 128-bit integer of weight 2^(64k - 1075);
//                  a term m * 2^(e' - 1075) adds m << (e' & 63) (< 2^116) to slot
//                  e' >> 6.  33 slots x 16 B = 528 B per lane, 16.9 KB per warp:
//                  12 warps per SM.  One LDS.128 + 4 adds + one STS.128.
//   96             slot k = signed 96-bit integer of weight 2^(32k - 1075) — the
//                  reference's chunk weight — as a u32 plane and an s64 plane;
//                  66 slots, 25.3 KB per warp: 8 warps per SM.
//
// Either way 2^11 of headroom absorbs 2047 terms per slot; each lane
// renormalises (carries upward) at most every 2016 terms.  e' = max(e, 1) and the
// implicit one is dropped for e == 0 (denormals, paper §small).
//
// Why not the reference's 4096 shared bins: 64-bit shared atomics compile to
// ATOMS.CAST.SPIN.64 CAS loops on sm_100a, random-bin read-modify-writes cost
// ~3.5x in bank conflicts, and narrow data (U[0,1)) puts half of all terms in
// one bin.  Lane privatisation removes all three.
//
// Kernels
//   exsum_sum_kernel        K1+K2+K3: persistent grid (1 CTA per SM), each warp
//                           streams a contiguous range with 256-bit loads
//                           (register double-buffered, L2 bulk prefetch ahead),
//                           lanes accumulate privately; the CTA combines its
//                           lanes into 67 chunk sums, REDG.ADD.64 into the
//                           workspace; the last CTA canonicalises, resolves
//                           Inf/NaN by first index, rounds.
//   exsum_segmented_kernel  K4: one warp per segment (dynamic), same inner loop,
//                           warp-local combine + round, one double per segment.
//   exsum_merge_kernel      K5: merge of k gathered partial records + round.

#include <cuda_runtime.h>
#include <stdint.h>

#include "exsum_b200.h"
#include "exsum_core.h"

#ifndef EXSUM_EXPERIMENT
#define EXSUM_EXPERIMENT 0
#endif
#ifndef EXSUM_SLOT_BITS
#define EXSUM_SLOT_BITS 96
#endif
#ifndef EXSUM_DECODE
#define EXSUM_DECODE 2  // 0: ALU-pipe decode, 1: FMA-pipe decode, 2: pipe-balanced
#endif
#ifndef EXSUM_HSPLIT
#define EXSUM_HSPLIT 0  // slot96: high word as two 32-bit planes (all accesses 32-bit)
#endif
#ifndef EXSUM_PIPE
#define EXSUM_PIPE 0  // 0 serial RMW, 1 store forwarding, 2 run merge (slot layout 96)
#endif
#if EXSUM_HSPLIT && (EXSUM_DECODE != 2 || EXSUM_PIPE != 0 || EXSUM_SLOT_BITS != 96)
#error "EXSUM_HSPLIT needs EXSUM_DECODE=2, EXSUM_PIPE=0, EXSUM_SLOT_BITS=96"
#endif

namespace exsum_b200 {
namespace dev {

// ---------------------------------------------------------------- workspace

// Zero-initialised global state of one (possibly multi-launch) accumulation.
// Special indices are stored bit-inverted so that 0 means "none" and the first
// occurrence wins under atomicMax.
struct Workspace {
  unsigned long long chunk[kChunks];
  unsigned long long inv_pinf, inv_ninf, inv_nan;
  unsigned long long nan_payload;
  unsigned int done;      // CTAs finished in the current launch
  unsigned int seg_next;  // segmented: next segment to claim
  unsigned int seg_done;  // segmented: warps finished
  unsigned int pad_;
};

struct Specials {                // first occurrences seen by one lane
  unsigned long long P, M, N;    // index (global or segment-local), ~0 = none
};

__device__ __forceinline__ uint32_t exponent_field(uint32_t hi) { return (hi >> 20) & 0x7FFu; }

// =========================================================== slot layout: 128
namespace slot128 {

constexpr int kWarps = 12;
constexpr int kSlots = 33;                  // 0..31 take terms (e' >> 6), 32 carries only
constexpr int kWarpSmem = kSlots * 32 * 16;  // 16,896 B
constexpr int kDefaultVec = 4;

struct Lane {
  uint4 *P;     // this lane's slot 0; slot k at P[32 k] (lane-interleaved 16 B entries)
  uint32_t sa;  // shared address of P; slot k at sa + 512 k
};

__device__ __forceinline__ Lane lane_view(unsigned char *warp_smem, int lane) {
  Lane v;
  v.P = reinterpret_cast<uint4 *>(warp_smem) + lane;
  v.sa = static_cast<uint32_t>(__cvta_generic_to_shared(v.P));
  return v;
}

// term = (-1)^s m 2^(e'-1075): add m << sh, sh = e' & 63, to slot e' >> 6.  For a
// negative term add ~(m << sh) + 1: the complement is folded into the funnel
// shifts (fill word s), the +1 is the carry-in (CC.CF = s & 1 from s + s).
// -0.0 adds 2^128, i.e. nothing.
__device__ __forceinline__ void add_term(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e) {
  const uint32_t ep = max(e, 1u);
  const uint32_t imp = e ? 0x100000u : 0u;
  const uint32_t s = static_cast<uint32_t>(static_cast<int32_t>(hi) >> 31);
  const uint32_t mx = ((hi & 0xFFFFFu) | imp) ^ s;
  const uint32_t lx = lo ^ s;
  const uint32_t w0 = __funnelshift_l(s, lx, ep);   // shift count taken mod 32
  const uint32_t w1 = __funnelshift_l(lx, mx, ep);
  const uint32_t w2 = __funnelshift_l(mx, s, ep);
  const bool up = (ep & 32u) != 0u;                  // shift by 32 more: one word up
  const uint32_t u0 = up ? s : w0, u1 = up ? w0 : w1, u2 = up ? w1 : w2, u3 = up ? w2 : s;
  const uint32_t addr = a.sa + ((ep >> 6) << 9);
  asm volatile(
      "{\n\t.reg .u32 q0, q1, q2, q3, cf;\n\t"
      "ld.shared.v4.u32 {q0, q1, q2, q3}, [%0];\n\t"
      "add.cc.u32 cf, %1, %1;\n\t"
      "addc.cc.u32 q0, q0, %2;\n\t"
      "addc.cc.u32 q1, q1, %3;\n\t"
      "addc.cc.u32 q2, q2, %4;\n\t"
      "addc.u32 q3, q3, %5;\n\t"
      "st.shared.v4.u32 [%0], {q0, q1, q2, q3};\n\t}"
      :
      : "r"(addr), "r"(s), "r"(u0), "r"(u1), "r"(u2), "r"(u3)
      : "memory");
}

// Carry upward: slots 0..31 end in [0, 2^64) (high half zero), slot 32 keeps the
// rest.  Each slot has absorbed <= 2047 terms (< 2^127 with the incoming carry).
__device__ __forceinline__ void normalize(const Lane &a) {
  long long c = 0;
#pragma unroll 4
  for (int k = 0; k < kSlots - 1; ++k) {
    const uint4 v = a.P[32 * k];
    const unsigned long long lo = (static_cast<unsigned long long>(v.y) << 32) | v.x;
    const long long hi = static_cast<long long>((static_cast<unsigned long long>(v.w) << 32) | v.z);
    const unsigned long long nlo = lo + static_cast<unsigned long long>(c);
    const long long nhi = hi + (c >> 63) + (nlo < lo ? 1 : 0);
    a.P[32 * k] = make_uint4(static_cast<uint32_t>(nlo), static_cast<uint32_t>(nlo >> 32), 0u, 0u);
    c = nhi;
  }
  const uint4 v = a.P[32 * (kSlots - 1)];
  const unsigned long long lo = (static_cast<unsigned long long>(v.y) << 32) | v.x;
  const long long hi = static_cast<long long>((static_cast<unsigned long long>(v.w) << 32) | v.z);
  const unsigned long long nlo = lo + static_cast<unsigned long long>(c);
  const unsigned long long nhi =
      static_cast<unsigned long long>(hi + (c >> 63) + (nlo < lo ? 1 : 0));
  a.P[32 * (kSlots - 1)] = make_uint4(static_cast<uint32_t>(nlo), static_cast<uint32_t>(nlo >> 32),
                                      static_cast<uint32_t>(nhi), static_cast<uint32_t>(nhi >> 32));
}

// The warp's exact sum as 67 chunk values (row[0..66], |row[i]| < 2^38):
// normalise each lane, then lane j sums slot j's two low words over all lanes.
__device__ __forceinline__ void warp_chunks(unsigned char *warp_smem, const Lane &a, int lane,
                                            long long *row) {
  normalize(a);
  __syncwarp();
  const uint4 *base = reinterpret_cast<const uint4 *>(warp_smem);
  unsigned long long s0 = 0, s1 = 0;
#pragma unroll 8
  for (int i = 0; i < 32; ++i) {
    const int col = (i + lane) & 31;
    const uint2 v = *reinterpret_cast<const uint2 *>(&base[lane * 32 + col]);
    s0 += v.x;
    s1 += v.y;
  }
  row[2 * lane] = static_cast<long long>(s0);
  row[2 * lane + 1] = static_cast<long long>(s1);
  const uint4 t = base[(kSlots - 1) * 32 + lane];
  unsigned long long c64 = t.x, c65 = t.y;
  long long c66 = static_cast<long long>((static_cast<unsigned long long>(t.w) << 32) | t.z);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    c64 += __shfl_xor_sync(0xffffffffu, c64, o);
    c65 += __shfl_xor_sync(0xffffffffu, c65, o);
    c66 += __shfl_xor_sync(0xffffffffu, c66, o);
  }
  if (lane == 0) {
    row[64] = static_cast<long long>(c64);
    row[65] = static_cast<long long>(c65);
    row[66] = c66;
  }
}

}  // namespace slot128

// ============================================================ slot layout: 96
namespace slot96 {

constexpr int kWarps = 8;
constexpr int kSlots = 66;       // slots 0..63 take terms (e' >> 5), 64..65 only carries
constexpr int kLPlane = kSlots * 32 * 4;
constexpr int kHPlane = kSlots * 32 * 8;
constexpr int kWarpSmem = kLPlane + kHPlane;  // 25,344 B
constexpr int kDefaultVec = 8;

// Slot k's low word is at sl + 128 k and its high word at 2 * (sl + 128 k) + hoff.
struct Lane {
  uint32_t *L;            // &Lplane[0][lane]; slot k at L[32 k]
  unsigned long long *H;  // &Hplane[0][lane]; slot k at H[32 k]
  uint32_t sl;
  uint32_t hoff;
  uint32_t two;   // 2 and 128, opaque to ptxas: keeps the address arithmetic
  uint32_t c128;  // IMADs on the FMA pipe instead of LEAs on the ALU pipe
};

__device__ __forceinline__ Lane lane_view(unsigned char *warp_smem, int lane) {
  Lane v;
  v.L = reinterpret_cast<uint32_t *>(warp_smem) + lane;
  v.H = reinterpret_cast<unsigned long long *>(warp_smem + kLPlane) + lane;
  v.sl = static_cast<uint32_t>(__cvta_generic_to_shared(v.L));
  v.hoff = static_cast<uint32_t>(__cvta_generic_to_shared(v.H)) - 2u * v.sl;
  v.two = (blockDim.x >> 30) + 2u;
  v.c128 = v.two * 64u;
  return v;
}

// Same scheme as slot128 with a 96-bit window: m << (e' & 31) at slot e' >> 5.
#if EXSUM_DECODE == 2
// Pipe-balanced form (the B200 integer ALU pipe and the FMA pipe each retire 16
// lanes/clk/SMSP; SHF/LOP3/IADD3/VIMNMX/ISETP go to the ALU, IMAD/VIADD to the
// FMA pipe).  Per term: 11 ALU + 9 FMA + 4 LSU.  e (exponent field) and s (sign
// mask) come precomputed from the batch decode.
// The term as three 32-bit words of its complemented, shifted significand
// (u2:u1:u0 = s ? ~(m << sh) : m << sh; the +1 of a negative term is the carry-in
// s + s), plus e' = max(e, 1).
__device__ __forceinline__ void decode96(uint32_t lo, uint32_t hi, uint32_t e, uint32_t &s,
                                         uint32_t &u0, uint32_t &u1, uint32_t &u2,
                                         uint32_t &ep) {
  uint32_t d, mhi, mh, m1, lx, mx;
  asm("shr.s32 %0, %1, 31;" : "=r"(s) : "r"(hi));                         // ALU: sign mask
  asm("max.u32 %0, %1, 1;" : "=r"(ep) : "r"(e));                         // ALU
  asm("mad.lo.u32 %0, %1, -1, %2;" : "=r"(d) : "r"(e), "r"(ep));          // FMA: 1 iff e == 0
  asm("lop3.b32 %0, %1, 0xFFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x100000u));  // ALU: (a&b)|c
  asm("mad.lo.u32 %0, %1, -1048576, %2;" : "=r"(mh) : "r"(d), "r"(mhi));  // FMA: drop implicit 1
  asm("mad.lo.u32 %0, %1, 2, 1;" : "=r"(m1) : "r"(s));                    // FMA: +-1
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(lx) : "r"(lo), "r"(m1), "r"(s));  // FMA: lo ^ s
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(mx) : "r"(mh), "r"(m1), "r"(s));  // FMA: mh ^ s
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u0) : "r"(s), "r"(lx), "r"(ep));   // ALU
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u1) : "r"(lx), "r"(mx), "r"(ep));  // ALU
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u2) : "r"(mx), "r"(s), "r"(ep));   // ALU
}

// Read-modify-write of slot k with a 96-bit two's-complement value (no carry-in).
__device__ __forceinline__ void slot_add96(const Lane &a, uint32_t k, uint32_t v0, uint32_t v1,
                                           uint32_t v2) {
  uint32_t la, ha;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(la) : "r"(k), "r"(a.c128), "r"(a.sl));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(ha) : "r"(la), "r"(a.two), "r"(a.hoff));
  asm volatile(
      "{\n\t.reg .u32 l, h0, h1;\n\t"
      "ld.shared.u32 l, [%0];\n\t"
      "ld.shared.v2.u32 {h0, h1}, [%1];\n\t"
      "add.cc.u32 l, l, %2;\n\t"
      "addc.cc.u32 h0, h0, %3;\n\t"
      "addc.u32 h1, h1, %4;\n\t"
      "st.shared.u32 [%0], l;\n\t"
      "st.shared.v2.u32 [%1], {h0, h1};\n\t}"
      :
      : "r"(la), "r"(ha), "r"(v0), "r"(v1), "r"(v2)
      : "memory");
}

__device__ __forceinline__ void add_term(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e) {
  uint32_t s, ep, k, la, ha, u0, u1, u2;
  decode96(lo, hi, e, s, u0, u1, u2, ep);
  asm("shr.u32 %0, %1, 5;" : "=r"(k) : "r"(ep));                          // ALU
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(la) : "r"(k), "r"(a.c128), "r"(a.sl));  // FMA
#if EXSUM_HSPLIT
  // three 32-bit planes: every access is a conflict-free 32-bit LDS/STS at
  // la + {0, kPlane, 2 kPlane} (immediate offsets, no second address)
  (void)ha;
  asm volatile(
      "{\n\t.reg .u32 l, h0, h1, cf;\n\t"
      "ld.shared.u32 l, [%0];\n\t"
      "ld.shared.u32 h0, [%0+8448];\n\t"
      "ld.shared.u32 h1, [%0+16896];\n\t"
      "add.cc.u32 cf, %1, %1;\n\t"
      "addc.cc.u32 l, l, %2;\n\t"
      "addc.cc.u32 h0, h0, %3;\n\t"
      "addc.u32 h1, h1, %4;\n\t"
      "st.shared.u32 [%0], l;\n\t"
      "st.shared.u32 [%0+8448], h0;\n\t"
      "st.shared.u32 [%0+16896], h1;\n\t}"
      :
      : "r"(la), "r"(s), "r"(u0), "r"(u1), "r"(u2)
      : "memory");
  return;
#endif
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(ha) : "r"(la), "r"(a.two), "r"(a.hoff));  // FMA
  asm volatile(
      "{\n\t.reg .u32 l, h0, h1, cf;\n\t"
      "ld.shared.u32 l, [%0];\n\t"
      "ld.shared.v2.u32 {h0, h1}, [%1];\n\t"
      "add.cc.u32 cf, %2, %2;\n\t"
      "addc.cc.u32 l, l, %3;\n\t"
      "addc.cc.u32 h0, h0, %4;\n\t"
      "addc.u32 h1, h1, %5;\n\t"
      "st.shared.u32 [%0], l;\n\t"
      "st.shared.v2.u32 [%1], {h0, h1};\n\t}"
      :
      : "r"(la), "r"(ha), "r"(s), "r"(u0), "r"(u1), "r"(u2)
      : "memory");
}
#else
__device__ __forceinline__ void add_term(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e) {
#if EXSUM_DECODE == 1
  // Decode on the FMA pipe (IMAD / IMAD.HI) to unload the integer ALU pipe:
  // t = hi >> 20, s = sign mask, low 20 mantissa bits = hi - t 2^20, implicit
  // one = (e + 2047) >> 11, x ^ s = x (2s + 1) + s for s in {0, -1}.
  const uint32_t t = __umulhi(hi, 4096u);
  const uint32_t s = static_cast<uint32_t>(__mulhi(static_cast<int>(hi), 1));
  const uint32_t ib = __umulhi(e + 2047u, 2097152u);
  const uint32_t mh = hi - t * 1048576u + ib * 1048576u;
  const uint32_t ep = max(e, 1u);
  const uint32_t m1 = s * 2u + 1u;
  const uint32_t lx = lo * m1 + s;
  const uint32_t mx = mh * m1 + s;
#else
  const uint32_t ep = max(e, 1u);
  const uint32_t imp = e ? 0x100000u : 0u;
  const uint32_t s = static_cast<uint32_t>(static_cast<int32_t>(hi) >> 31);
  const uint32_t mx = ((hi & 0xFFFFFu) | imp) ^ s;
  const uint32_t lx = lo ^ s;
#endif
  const uint32_t u0 = __funnelshift_l(s, lx, ep);
  const uint32_t u1 = __funnelshift_l(lx, mx, ep);
  const uint32_t u2 = __funnelshift_l(mx, s, ep);
  const uint32_t la = a.sl + ((ep >> 5) << 7);
  const uint32_t ha = 2u * la + a.hoff;
  asm volatile(
      "{\n\t.reg .u32 l, h0, h1, cf;\n\t"
      "ld.shared.u32 l, [%0];\n\t"
      "ld.shared.v2.u32 {h0, h1}, [%1];\n\t"
      "add.cc.u32 cf, %2, %2;\n\t"
      "addc.cc.u32 l, l, %3;\n\t"
      "addc.cc.u32 h0, h0, %4;\n\t"
      "addc.u32 h1, h1, %5;\n\t"
      "st.shared.u32 [%0], l;\n\t"
      "st.shared.v2.u32 [%1], {h0, h1};\n\t}"
      :
      : "r"(la), "r"(ha), "r"(s), "r"(u0), "r"(u1), "r"(u2)
      : "memory");
}
#endif

// Carry upward: L_k in [0, 2^32), H_k = 0 for k < 65; slot 65 keeps the rest.
#if EXSUM_HSPLIT
__device__ __forceinline__ void normalize(const Lane &a) {
  uint32_t *H0 = a.L + kSlots * 32, *H1 = a.L + 2 * kSlots * 32;
  long long c = 0;
#pragma unroll 6
  for (int k = 0; k < kSlots - 1; ++k) {
    const long long u = static_cast<long long>(a.L[32 * k]) + c;
    const long long h = static_cast<long long>((static_cast<unsigned long long>(H1[32 * k]) << 32) | H0[32 * k]);
    a.L[32 * k] = static_cast<uint32_t>(u);
    H0[32 * k] = 0u;
    H1[32 * k] = 0u;
    c = h + (u >> 32);
  }
  const int k = kSlots - 1;
  const long long u = static_cast<long long>(a.L[32 * k]) + c;
  const long long h = static_cast<long long>((static_cast<unsigned long long>(H1[32 * k]) << 32) | H0[32 * k]);
  const unsigned long long nh = static_cast<unsigned long long>(h + (u >> 32));
  a.L[32 * k] = static_cast<uint32_t>(u);
  H0[32 * k] = static_cast<uint32_t>(nh);
  H1[32 * k] = static_cast<uint32_t>(nh >> 32);
}
#else
__device__ __forceinline__ void normalize(const Lane &a) {
  long long c = 0;
#pragma unroll 6
  for (int k = 0; k < kSlots - 1; ++k) {
    const long long u = static_cast<long long>(a.L[32 * k]) + c;
    const long long h = static_cast<long long>(a.H[32 * k]);
    a.L[32 * k] = static_cast<uint32_t>(u);
    a.H[32 * k] = 0ull;
    c = h + (u >> 32);
  }
  const int k = kSlots - 1;
  const long long u = static_cast<long long>(a.L[32 * k]) + c;
  a.L[32 * k] = static_cast<uint32_t>(u);
  a.H[32 * k] = static_cast<unsigned long long>(static_cast<long long>(a.H[32 * k]) + (u >> 32));
}
#endif

// ---- pipelined term streams (EXSUM_PIPE) ------------------------------------
//
// add_term above is a strict read-modify-write chain per lane: the next term's
// LDS cannot issue before this term's STS.  The pipes break that chain.
//
// Forward (EXSUM_PIPE 1): term j's LDS is issued before term j-1's STS; if both
// hit the same slot, j-1's fresh value is forwarded from registers.
// Merge (EXSUM_PIPE 2): a "pending" slot accumulates consecutive terms that hit
// it in registers; only when the slot changes is the pending value committed
// (predicated STS) and the new slot loaded (predicated LDS, issued before the
// commit).  Narrow exponent ranges then touch shared memory rarely.

struct Pipe {
  uint32_t pla;         // L-plane address of the pending slot
  uint32_t v0, v1, v2;  // forward: its new value; merge: its loaded base value
  uint32_t a0, a1, a2;  // merge: pending addend
};

__device__ __forceinline__ void term_words(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e,
                                           uint32_t &s, uint32_t &u0, uint32_t &u1,
                                           uint32_t &u2, uint32_t &la) {
  const uint32_t ep = max(e, 1u);
  const uint32_t imp = e ? 0x100000u : 0u;
  s = static_cast<uint32_t>(static_cast<int32_t>(hi) >> 31);
  const uint32_t mx = ((hi & 0xFFFFFu) | imp) ^ s;
  const uint32_t lx = lo ^ s;
  u0 = __funnelshift_l(s, lx, ep);
  u1 = __funnelshift_l(lx, mx, ep);
  u2 = __funnelshift_l(mx, s, ep);
  la = a.sl + ((ep >> 5) << 7);
}

__device__ __forceinline__ void pipe_init(const Lane &a, Pipe &p) {
  p.pla = a.sl;  // slot 0
  const uint32_t ha = 2u * p.pla + a.hoff;
  asm volatile("ld.shared.u32 %0, [%3];\n\tld.shared.v2.u32 {%1, %2}, [%4];"
               : "=r"(p.v0), "=r"(p.v1), "=r"(p.v2)
               : "r"(p.pla), "r"(ha)
               : "memory");
  p.a0 = p.a1 = p.a2 = 0u;
}

__device__ __forceinline__ void pipe_flush(const Lane &a, Pipe &p) {
  uint32_t c0 = p.v0, c1 = p.v1, c2 = p.v2;
#if EXSUM_PIPE == 2
  asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
      : "+r"(c0), "+r"(c1), "+r"(c2)
      : "r"(p.a0), "r"(p.a1), "r"(p.a2));
#endif
  const uint32_t ha = 2u * p.pla + a.hoff;
  asm volatile("st.shared.u32 [%0], %2;\n\tst.shared.v2.u32 [%1], {%3, %4};" ::"r"(p.pla),
               "r"(ha), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

__device__ __forceinline__ void pipe_step(const Lane &a, Pipe &p, uint32_t lo, uint32_t hi,
                                          uint32_t e) {
  uint32_t s, u0, u1, u2, la;
  term_words(a, lo, hi, e, s, u0, u1, u2, la);
  const uint32_t ha = 2u * la + a.hoff;
  const uint32_t pha = 2u * p.pla + a.hoff;
#if EXSUM_PIPE == 1
  uint32_t l0, l1, l2;
  asm volatile(
      "ld.shared.u32 %0, [%3];\n\t"
      "ld.shared.v2.u32 {%1, %2}, [%4];\n\t"
      "st.shared.u32 [%5], %7;\n\t"
      "st.shared.v2.u32 [%6], {%8, %9};"
      : "=r"(l0), "=r"(l1), "=r"(l2)
      : "r"(la), "r"(ha), "r"(p.pla), "r"(pha), "r"(p.v0), "r"(p.v1), "r"(p.v2)
      : "memory");
  const bool same = la == p.pla;
  uint32_t n0 = same ? p.v0 : l0, n1 = same ? p.v1 : l1, n2 = same ? p.v2 : l2;
  asm("{\n\t.reg .u32 cf;\n\tadd.cc.u32 cf, %3, %3;\n\taddc.cc.u32 %0, %0, %4;\n\t"
      "addc.cc.u32 %1, %1, %5;\n\taddc.u32 %2, %2, %6;\n\t}"
      : "+r"(n0), "+r"(n1), "+r"(n2)
      : "r"(s), "r"(u0), "r"(u1), "r"(u2));
  p.v0 = n0;
  p.v1 = n1;
  p.v2 = n2;
  p.pla = la;
#else
  // commit value of the pending slot (used only if the slot changes)
  uint32_t c0 = p.v0, c1 = p.v1, c2 = p.v2;
  asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
      : "+r"(c0), "+r"(c1), "+r"(c2)
      : "r"(p.a0), "r"(p.a1), "r"(p.a2));
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, %5;\n\t"
      "@q ld.shared.u32 %0, [%3];\n\t"
      "@q ld.shared.v2.u32 {%1, %2}, [%4];\n\t"
      "@q st.shared.u32 [%5], %7;\n\t"
      "@q st.shared.v2.u32 [%6], {%8, %9};\n\t}"
      : "+r"(p.v0), "+r"(p.v1), "+r"(p.v2)
      : "r"(la), "r"(ha), "r"(p.pla), "r"(pha), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
  const bool same = la == p.pla;
  uint32_t n0 = same ? p.a0 : 0u, n1 = same ? p.a1 : 0u, n2 = same ? p.a2 : 0u;
  asm("{\n\t.reg .u32 cf;\n\tadd.cc.u32 cf, %3, %3;\n\taddc.cc.u32 %0, %0, %4;\n\t"
      "addc.cc.u32 %1, %1, %5;\n\taddc.u32 %2, %2, %6;\n\t}"
      : "+r"(n0), "+r"(n1), "+r"(n2)
      : "r"(s), "r"(u0), "r"(u1), "r"(u2));
  p.a0 = n0;
  p.a1 = n1;
  p.a2 = n2;
  p.pla = la;
#endif
}

// The warp's exact sum as 67 chunk values, straight from the (unnormalised)
// slots: slot k = L_k + 2^32 H_k feeds chunk k (L_k), chunk k+1 (low word of H_k)
// and chunk k+2 (signed high word of H_k); every addend is < 2^32 in magnitude,
// so 32-lane sums stay below 2^38.  The high word of the carry-only slot 65
// belongs to chunk 67 and is folded into chunk 66.  Reads are bank-skewed.
__device__ __forceinline__ void warp_chunks(unsigned char *warp_smem, const Lane &a, int lane,
                                            long long *row) {
  (void)a;
  __syncwarp();
  const uint32_t *Lp = reinterpret_cast<const uint32_t *>(warp_smem);
#if EXSUM_HSPLIT
  const uint32_t *H0 = Lp + kSlots * 32, *H1 = Lp + 2 * kSlots * 32;
#define EXSUM_HLO(k, col) H0[(k) * 32 + (col)]
#define EXSUM_HHI(k, col) H1[(k) * 32 + (col)]
#else
  const uint32_t *Hw = reinterpret_cast<const uint32_t *>(warp_smem + kLPlane);  // H as 2 words
#define EXSUM_HLO(k, col) Hw[2 * ((k) * 32 + (col))]
#define EXSUM_HHI(k, col) Hw[2 * ((k) * 32 + (col)) + 1]
#endif
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int c = 32 * r + lane;  // chunk index this lane sums
    if (c >= kChunks) break;
    long long acc = 0;
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
      const int col = (i + lane) & 31;
      if (c < kSlots) acc += Lp[c * 32 + col];
      if (c >= 1) acc += EXSUM_HLO(c - 1, col);  // low word of H_{c-1}
      if (c >= 2 && c - 2 < kSlots - 1)
        acc += static_cast<int32_t>(EXSUM_HHI(c - 2, col));  // high word of H_{c-2}
      if (c == kChunks - 1)
        acc += static_cast<long long>(static_cast<int32_t>(EXSUM_HHI(kSlots - 1, col)))
               << 32;  // high word of H_65 (chunk 67) folded into chunk 66
    }
#undef EXSUM_HLO
#undef EXSUM_HHI
    row[c] = acc;
  }
}

}  // namespace slot96

#if EXSUM_SLOT_BITS == 96
namespace acc = slot96;
#elif EXSUM_SLOT_BITS == 128
namespace acc = slot128;
#else
#error "EXSUM_SLOT_BITS must be 96 or 128"
#endif

// ------------------------------------------------------------ common machinery

constexpr int kWarps = acc::kWarps;
constexpr int kThreads = kWarps * 32;
constexpr int kWarpSmem = acc::kWarpSmem;
#ifndef EXSUM_VEC_PER_LANE
#define EXSUM_VEC_PER_LANE acc::kDefaultVec
#endif
constexpr int kVecPerLane = EXSUM_VEC_PER_LANE;   // 256-bit vectors per lane per batch
constexpr int kBatchTerms = kVecPerLane * 4;
constexpr int kNormEvery = 2016 / kBatchTerms;    // batches between renormalisations
#ifndef EXSUM_PREFETCH_BATCHES
#define EXSUM_PREFETCH_BATCHES 1
#endif
constexpr int kPrefetchBatches = EXSUM_PREFETCH_BATCHES;  // L2 prefetch distance
#ifndef EXSUM_UNIFORM_FAST
#define EXSUM_UNIFORM_FAST 1  // register fast path when a warp's batch hits one slot per lane
#endif
#ifndef EXSUM_UNIFORM_BACKOFF
#define EXSUM_UNIFORM_BACKOFF 7
#endif
constexpr int kUniformBackoff = EXSUM_UNIFORM_BACKOFF;
#ifndef EXSUM_ROLL
#define EXSUM_ROLL 1  // rolling single-buffer loads with batch-end Inf/NaN fix-up
#endif
#ifndef EXSUM_CHECK_GROUP
#define EXSUM_CHECK_GROUP 0  // vectors per Inf/NaN-check group (0: whole batch)
#endif
#ifndef EXSUM_PREFETCH_LANES
#define EXSUM_PREFETCH_LANES 0
#endif
#ifndef EXSUM_BUFFERS
#define EXSUM_BUFFERS 1  // register batch buffers (1: rely on the L2 prefetch)
#endif
constexpr int kScratch = kWarps * kChunks * 8;              // per-warp chunk rows
constexpr int kSmem = kWarps * kWarpSmem + kScratch;
static_assert(kSmem <= 227 * 1024, "shared memory budget");
static_assert(kNormEvery >= 1, "batch too large for the carry budget");

using acc::Lane;

// Term stream over a lane accumulator: pipelined (EXSUM_PIPE) or plain RMW.
#if EXSUM_PIPE != 0 && EXSUM_SLOT_BITS == 96
using acc::Pipe;
__device__ __forceinline__ void stream_begin(const Lane &a, Pipe &p) { acc::pipe_init(a, p); }
__device__ __forceinline__ void stream_end(const Lane &a, Pipe &p) { acc::pipe_flush(a, p); }
__device__ __forceinline__ void stream_term(const Lane &a, Pipe &p, uint32_t lo, uint32_t hi,
                                            uint32_t e) {
  acc::pipe_step(a, p, lo, hi, e);
}
#else
struct Pipe {};
__device__ __forceinline__ void stream_begin(const Lane &, Pipe &) {}
__device__ __forceinline__ void stream_end(const Lane &, Pipe &) {}
__device__ __forceinline__ void stream_term(const Lane &a, Pipe &, uint32_t lo, uint32_t hi,
                                            uint32_t e) {
  acc::add_term(a, lo, hi, e);
}
#endif

// Zero one warp's accumulator cooperatively with 16-byte stores.
__device__ __forceinline__ void zero_warp(unsigned char *warp_smem, int lane) {
  uint4 *p = reinterpret_cast<uint4 *>(warp_smem);
  constexpr int n16 = kWarpSmem / 16;
#pragma unroll 4
  for (int i = lane; i < n16; i += 32) p[i] = make_uint4(0, 0, 0, 0);
}

__device__ __forceinline__ void record_special(Specials &sp, uint32_t lo, uint32_t hi,
                                               unsigned long long index) {
  if ((hi & 0xFFFFFu) | lo) {
    sp.N = min(sp.N, index);
  } else if (hi >> 31) {
    sp.M = min(sp.M, index);
  } else {
    sp.P = min(sp.P, index);
  }
}

// One term of a scalar head/tail: Inf/NaN recorded, everything else added.
__device__ __forceinline__ void add_term_checked(const Lane &a, Specials &sp, uint32_t lo,
                                                 uint32_t hi, unsigned long long index) {
  const uint32_t e = exponent_field(hi);
  if (e == 0x7FFu) {
    record_special(sp, lo, hi, index);
  } else {
    acc::add_term(a, lo, hi, e);
  }
}

// 256-bit streaming load (LDG.E.NA.ENL2.256): 4 terms per lane per instruction.
__device__ __forceinline__ void ldg256(const double *p, uint32_t (&w)[8]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7])
      : "l"(p));
}

struct Batch {
  uint32_t w[kVecPerLane][8];
};

// Load one batch: vectors v0 + u*32 + lane (u < kVecPerLane) of the 32-byte
// vector array starting at X4; vectors at or beyond vend read as zero terms.
__device__ __forceinline__ void load_batch(Batch &b, const double *X4, long long v0,
                                           long long vend, int lane) {
  if (v0 + kVecPerLane * 32 <= vend) {
#pragma unroll
    for (int u = 0; u < kVecPerLane; ++u) ldg256(X4 + 4 * (v0 + u * 32 + lane), b.w[u]);
  } else {
#pragma unroll
    for (int u = 0; u < kVecPerLane; ++u) {
      const long long v = v0 + u * 32 + lane;
#pragma unroll
      for (int q = 0; q < 8; ++q) b.w[u][q] = 0u;
      if (v < vend) ldg256(X4 + 4 * v, b.w[u]);
    }
  }
}

// Bulk L2 prefetch (cp.async.bulk.prefetch.L2) of one batch-sized stretch of
// 32-byte vectors starting at vector v0, clipped to vend.  Issued by one lane a
// few batches ahead of the register loads; costs no registers, no shared memory.
__device__ __forceinline__ void prefetch_l2(const double *X4, long long v0, long long vend) {
#if EXSUM_PREFETCH_LANES
  // per-lane variant: every lane prefetches the 256 B of its own vectors
  (void)vend;
  return;
#endif
  if (v0 >= vend) return;
  long long nv = vend - v0;
  if (nv > kVecPerLane * 32) nv = kVecPerLane * 32;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(X4 + 4 * v0),
               "r"(static_cast<uint32_t>(nv * 32))
               : "memory");
}

// Process one batch (kBatchTerms terms per lane).  index_of_vec0 is the
// special-value index of term 0 of the batch's first vector.
#if EXSUM_CHECK_GROUP > 0 && EXSUM_EXPERIMENT == 0
// Grouped form: the Inf/NaN test and the adds run per group of G vectors, so the
// first group is processed while the batch's later loads are still in flight.
__device__ __forceinline__ void process_batch(const Lane &a, Pipe &pp, Specials &sp, Batch &b,
                                              int lane, unsigned long long index_of_vec0) {
  constexpr int G = EXSUM_CHECK_GROUP;
  static_assert(kVecPerLane % G == 0, "group must divide the batch");
#pragma unroll
  for (int g = 0; g < kVecPerLane; g += G) {
    uint32_t e[G][4];
    uint32_t emax = 0;
#pragma unroll
    for (int u = 0; u < G; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        e[u][q] = exponent_field(b.w[g + u][2 * q + 1]);
        emax = max(emax, e[u][q]);
      }
    if (emax == 0x7FFu) {  // rare: record Inf/NaN and turn them into zero terms
#pragma unroll
      for (int u = 0; u < G; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (e[u][q] == 0x7FFu) {
            record_special(sp, b.w[g + u][2 * q], b.w[g + u][2 * q + 1],
                           index_of_vec0 + 4ull * static_cast<unsigned long long>((g + u) * 32 + lane) + q);
            b.w[g + u][2 * q] = 0u;
            b.w[g + u][2 * q + 1] = 0u;
            e[u][q] = 0u;
          }
    }
#pragma unroll
    for (int u = 0; u < G; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        stream_term(a, pp, b.w[g + u][2 * q], b.w[g + u][2 * q + 1], e[u][q]);
  }
}
#else
__device__ __forceinline__ void process_batch(const Lane &a, Pipe &pp, Specials &sp, Batch &b,
                                              int lane, unsigned long long index_of_vec0) {
  uint32_t e[kVecPerLane][4];
  bool special = false;
#if EXSUM_DECODE == 2
  // exponent fields; "any Inf/NaN" = (max exponent == 2047), 3-input max chains
  uint32_t emax = 0;
#pragma unroll
  for (int u = 0; u < kVecPerLane; ++u)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      e[u][q] = exponent_field(b.w[u][2 * q + 1]);
      emax = max(emax, e[u][q]);
    }
  special = emax == 0x7FFu;
#else
#pragma unroll
  for (int u = 0; u < kVecPerLane; ++u)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#if EXSUM_DECODE == 1
      {
        const uint32_t hw = b.w[u][2 * q + 1];
        e[u][q] = __umulhi(hw, 4096u) + static_cast<uint32_t>(__mulhi(static_cast<int>(hw), 1)) * 2048u;
      }
#else
      e[u][q] = exponent_field(b.w[u][2 * q + 1]);
#endif
      special |= e[u][q] == 0x7FFu;
    }
#endif
  if (special) {  // rare: record Inf/NaN and turn them into zero terms
#pragma unroll
    for (int u = 0; u < kVecPerLane; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (e[u][q] == 0x7FFu) {
          record_special(sp, b.w[u][2 * q], b.w[u][2 * q + 1],
                         index_of_vec0 + 4ull * static_cast<unsigned long long>(u * 32 + lane) + q);
          b.w[u][2 * q] = 0u;
          b.w[u][2 * q + 1] = 0u;
          e[u][q] = 0u;
        }
  }
#if EXSUM_EXPERIMENT == 0
#pragma unroll
  for (int u = 0; u < kVecPerLane; ++u)
#pragma unroll
    for (int q = 0; q < 4; ++q) stream_term(a, pp, b.w[u][2 * q], b.w[u][2 * q + 1], e[u][q]);
#else
  // Tuning experiments only (wrong sums): 1 = same per-term ALU work, register
  // accumulation, one shared RMW per batch; 2 = loads only.
  uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
  for (int u = 0; u < kVecPerLane; ++u)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t lo = b.w[u][2 * q], hi = b.w[u][2 * q + 1];
#if EXSUM_EXPERIMENT == 1
      const uint32_t ep = max(e[u][q], 1u);
      const uint32_t imp = e[u][q] ? 0x100000u : 0u;
      const uint32_t s = static_cast<uint32_t>(static_cast<int32_t>(hi) >> 31);
      const uint32_t mx = ((hi & 0xFFFFFu) | imp) ^ s;
      const uint32_t lx = lo ^ s;
      const uint32_t w0 = __funnelshift_l(s, lx, ep), w1 = __funnelshift_l(lx, mx, ep);
      const uint32_t w2 = __funnelshift_l(mx, s, ep);
      asm("add.cc.u32 %0, %0, %4;\n\taddc.cc.u32 %1, %1, %5;\n\taddc.cc.u32 %2, %2, %6;\n\taddc.u32 %3, %3, %7;"
          : "+r"(r0), "+r"(r1), "+r"(r2), "+r"(r3) : "r"(w0), "r"(w1), "r"(w2), "r"(ep));
#else
      r0 ^= lo;
      r1 ^= hi;
#endif
    }
  acc::add_term(a, r0 ^ r2, r1 ^ r3, 5u);
#endif
}
#endif

// Accumulate x[begin, end) into the calling warp's lane accumulators.
// index_base is added to positions to form special-value indices; norm_count
// counts batches since the last renormalisation (warp-uniform).
__device__ void warp_accumulate(const double *__restrict__ x, unsigned long long begin,
                                unsigned long long end, unsigned long long index_base,
                                const Lane &a, Specials &sp, int &norm_count, int lane) {
  if (begin >= end) return;
  // Scalar head up to 32-byte alignment of &x[pos], scalar tail after the vectors.
  const uintptr_t addr = reinterpret_cast<uintptr_t>(x + begin);
  unsigned long long head = ((32u - (addr & 31u)) & 31u) >> 3;
  if (head > end - begin) head = end - begin;
  const unsigned long long *xb = reinterpret_cast<const unsigned long long *>(x);
  if (lane < static_cast<int>(head)) {
    const unsigned long long bits = __ldg(xb + begin + lane);
    add_term_checked(a, sp, static_cast<uint32_t>(bits), static_cast<uint32_t>(bits >> 32),
                     index_base + begin + lane);
  }
  const unsigned long long vbeg_t = begin + head;  // first vector's term position
  const long long nvec = static_cast<long long>((end - vbeg_t) >> 2);
  const double *X4 = x + vbeg_t;                   // 32-byte aligned
  const unsigned long long tail_t = vbeg_t + 4ull * static_cast<unsigned long long>(nvec);
  if (lane < static_cast<int>(end - tail_t)) {
    const unsigned long long bits = __ldg(xb + tail_t + lane);
    add_term_checked(a, sp, static_cast<uint32_t>(bits), static_cast<uint32_t>(bits >> 32),
                     index_base + tail_t + lane);
  }
  if (nvec <= 0) return;
  constexpr long long kStep = kVecPerLane * 32;
#if EXSUM_ROLL
  // Rolling single buffer: after a vector's four terms are added, its registers
  // are immediately refilled with the same vector of the next batch, so every
  // load is in flight for almost a whole batch without a second register set.
  // Inf/NaN: terms are added unconditionally; if the batch's maximum exponent
  // field is 2047 the batch is re-read and each Inf/NaN term is recorded and
  // its (garbage) contribution cancelled by adding its sign-flipped twin — exact
  // in the modular slot arithmetic, and before any renormalisation.
  Batch b0;
  const unsigned long long ib = index_base + vbeg_t;
  if (lane == 0) {
    for (int d = 0; d <= kPrefetchBatches; ++d) prefetch_l2(X4, d * kStep, nvec);
  }
  load_batch(b0, X4, 0, nvec, lane);
  int backoff = 0;
  for (long long v = 0; v < nvec; v += kStep) {
    const long long nv = v + kStep;
    if (lane == 0) prefetch_l2(X4, v + (kPrefetchBatches + 1) * kStep, nvec);
    uint32_t emax = 0;
    if (nv + kStep <= nvec) {
      // steady state: the next batch is complete, unguarded loads at immediate
      // offsets from one pointer
      const double *pn = X4 + 4 * (nv + lane);
#if EXSUM_UNIFORM_FAST
      // Slot of a term = top six exponent bits (hi bits 25..30; e = 0 maps to
      // slot 0 like e' = 1).  All terms of the batch share a slot iff the AND and
      // the OR of their high words agree on those bits: 3-input LOP3 chains, no
      // per-term exponent kept live.  Slot 63 may hold Inf/NaN: never "uniform".
      // Wide data rarely turns uniform: after a non-uniform batch the test is
      // skipped for the next kUniformBackoff batches (warp-uniform counter).
      bool fast = false;
      uint32_t kbits = 0u;
      if (backoff > 0) {
        --backoff;
      } else {
        uint32_t hor = 0u, hand = 0xFFFFFFFFu;
#pragma unroll
        for (int u = 0; u < kVecPerLane; ++u)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            hor |= b0.w[u][2 * q + 1];
            hand &= b0.w[u][2 * q + 1];
          }
        kbits = hor & 0x7E000000u;
        const bool uniform = kbits == (hand & 0x7E000000u) && kbits != 0x7E000000u;
        fast = __all_sync(0xffffffffu, uniform);
        if (!fast) backoff = kUniformBackoff;
      }
      if (fast) {
        // every lane's batch lies in one slot: sum it in registers (|sum| < 2^89),
        // then one read-modify-write of that slot
        uint32_t r0 = 0, r1 = 0, r2 = 0;
#pragma unroll
        for (int u = 0; u < kVecPerLane; ++u) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t sg, u0, u1, u2, ep;
            acc::decode96(b0.w[u][2 * q], b0.w[u][2 * q + 1], exponent_field(b0.w[u][2 * q + 1]),
                          sg, u0, u1, u2, ep);
            asm("{\n\t.reg .u32 cf;\n\tadd.cc.u32 cf, %3, %3;\n\taddc.cc.u32 %0, %0, %4;\n\t"
                "addc.cc.u32 %1, %1, %5;\n\taddc.u32 %2, %2, %6;\n\t}"
                : "+r"(r0), "+r"(r1), "+r"(r2)
                : "r"(sg), "r"(u0), "r"(u1), "r"(u2));
          }
          ldg256(pn + 4 * 32 * u, b0.w[u]);
        }
        acc::slot_add96(a, kbits >> 25, r0, r1, r2);
      } else {
#pragma unroll
        for (int u = 0; u < kVecPerLane; ++u) {
          uint32_t e[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            e[q] = exponent_field(b0.w[u][2 * q + 1]);
            emax = max(emax, e[q]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) acc::add_term(a, b0.w[u][2 * q], b0.w[u][2 * q + 1], e[q]);
          ldg256(pn + 4 * 32 * u, b0.w[u]);
        }
      }
#else
#pragma unroll
      for (int u = 0; u < kVecPerLane; ++u) {
        uint32_t e[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          e[q] = exponent_field(b0.w[u][2 * q + 1]);
          emax = max(emax, e[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) acc::add_term(a, b0.w[u][2 * q], b0.w[u][2 * q + 1], e[q]);
        ldg256(pn + 4 * 32 * u, b0.w[u]);
      }
#endif
    } else {
#pragma unroll
      for (int u = 0; u < kVecPerLane; ++u) {
        uint32_t e[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          e[q] = exponent_field(b0.w[u][2 * q + 1]);
          emax = max(emax, e[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) acc::add_term(a, b0.w[u][2 * q], b0.w[u][2 * q + 1], e[q]);
        const long long vv = nv + u * 32 + lane;
        if (vv < nvec) {
          ldg256(X4 + 4 * vv, b0.w[u]);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) b0.w[u][q] = 0u;
        }
      }
    }
    if (__builtin_expect(emax == 0x7FFu, 0)) {
      const unsigned long long *xb = reinterpret_cast<const unsigned long long *>(X4);
      for (int u = 0; u < kVecPerLane; ++u) {
        const long long vec = v + u * 32 + lane;
        if (vec >= nvec) break;
        for (int q = 0; q < 4; ++q) {
          const unsigned long long bits = __ldcg(xb + 4 * vec + q);
          const uint32_t lo = static_cast<uint32_t>(bits), hi = static_cast<uint32_t>(bits >> 32);
          if (exponent_field(hi) == 0x7FFu) {
            record_special(sp, lo, hi, ib + 4ull * static_cast<unsigned long long>(vec) + q);
            acc::add_term(a, lo, hi ^ 0x80000000u, 0x7FFu);  // cancel the garbage add
          }
        }
      }
    }
    if (++norm_count >= kNormEvery) {
      acc::normalize(a);
      norm_count = 0;
    }
  }
#elif EXSUM_BUFFERS == 1
  // Single register buffer: the L2 bulk prefetch (kPrefetchBatches ahead) hides
  // DRAM latency, the register load only waits for L2; frees 32-64 registers
  // for instruction-level parallelism.
  Batch b0;
  const unsigned long long ib = index_base + vbeg_t;
  if (lane == 0) {
    for (int d = 0; d <= kPrefetchBatches; ++d) prefetch_l2(X4, d * kStep, nvec);
  }
  Pipe pp;
  stream_begin(a, pp);
  for (long long v = 0; v < nvec; v += kStep) {
    load_batch(b0, X4, v, nvec, lane);
#if EXSUM_PREFETCH_LANES
    {
      const long long pv = v + (kPrefetchBatches + 1) * kStep;
#pragma unroll
      for (int u = 0; u < kVecPerLane; u += 4) {
        const long long q = pv + u * 32 + lane * 4;  // 4 consecutive vectors = 128 B
        if (q < nvec) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(X4 + 4 * q));
      }
    }
#else
    if (lane == 0) prefetch_l2(X4, v + (kPrefetchBatches + 1) * kStep, nvec);
#endif
    process_batch(a, pp, sp, b0, lane, ib + 4ull * static_cast<unsigned long long>(v));
    if (++norm_count >= kNormEvery) {
      stream_end(a, pp);
      acc::normalize(a);
      stream_begin(a, pp);
      norm_count = 0;
    }
  }
  stream_end(a, pp);
#else
  Batch b0, b1;
  long long v = 0;
  if (kPrefetchBatches > 0 && lane == 0) {
    for (int d = 1; d <= kPrefetchBatches; ++d) prefetch_l2(X4, d * kStep, nvec);
  }
  load_batch(b0, X4, 0, nvec, lane);
  const unsigned long long ib = index_base + vbeg_t;
  Pipe pp;
  stream_begin(a, pp);
  while (true) {
    long long nx = v + kStep;
    if (kPrefetchBatches > 0 && lane == 0) prefetch_l2(X4, v + (kPrefetchBatches + 1) * kStep, nvec);
    if (nx < nvec) load_batch(b1, X4, nx, nvec, lane);
    process_batch(a, pp, sp, b0, lane, ib + 4ull * static_cast<unsigned long long>(v));
    if (++norm_count >= kNormEvery) {
      stream_end(a, pp);
      acc::normalize(a);
      stream_begin(a, pp);
      norm_count = 0;
    }
    v = nx;
    if (v >= nvec) break;
    nx = v + kStep;
    if (kPrefetchBatches > 0 && lane == 0) prefetch_l2(X4, v + (kPrefetchBatches + 1) * kStep, nvec);
    if (nx < nvec) load_batch(b0, X4, nx, nvec, lane);
    process_batch(a, pp, sp, b1, lane, ib + 4ull * static_cast<unsigned long long>(v));
    if (++norm_count >= kNormEvery) {
      stream_end(a, pp);
      acc::normalize(a);
      stream_begin(a, pp);
      norm_count = 0;
    }
    v = nx;
    if (v >= nvec) break;
  }
  stream_end(a, pp);
#endif
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// Warp-parallel finalisation (all 32 lanes of one warp): the same canonical form
// and rounding as emit_record / exsum_core.h, without a 67-step serial chain.
//   1. carry propagation by repeated shuffle passes until no lane holds a carry
//      (two or three passes for accumulated chunk sums);
//   2. canonical top / fold of a -1 top chunk via ballots;
//   3. magnitude digits of a negative value by the two's-complement rule
//      (zero below the lowest nonzero digit z, -d_z at z, ~d_i above);
//   4. lane 0 rounds a 3-digit window at the leading digit with a sticky ballot.
// row: 67 chunk values in shared memory (any representation with |c| < 2^62).
__device__ void warp_emit(const long long *row, unsigned long long P, unsigned long long M,
                          unsigned long long N, unsigned long long payload, double *result,
                          exsum_partial *partial, int lane) {
  const unsigned FULL = 0xffffffffu;
  long long v[3];
  v[0] = row[lane];
  v[1] = row[lane + 32];
  v[2] = lane < 3 ? row[lane + 64] : 0;
  // 1. carries: chunk i keeps its low 32 bits, passes the rest to i + 1; chunk 66 keeps all.
  while (true) {
    long long c[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) c[r] = (32 * r + lane < kChunks - 1) ? (v[r] >> 32) : 0;
    if (!__any_sync(FULL, (c[0] | c[1] | c[2]) != 0)) break;
    long long in[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const long long up = __shfl_up_sync(FULL, c[r], 1);
      const long long wrap = r ? __shfl_sync(FULL, c[r - 1], 31) : 0;
      in[r] = lane ? up : wrap;
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int idx = 32 * r + lane;
      if (idx < kChunks - 1) v[r] &= 0xFFFFFFFFll;
      if (idx < kChunks) v[r] += in[r];
    }
  }
  const long long d66 = __shfl_sync(FULL, v[2], 2);
  // 2. canonical top.
  auto top_of = [&](unsigned b0, unsigned b1, unsigned b2) -> int {
    if (b2) return 64 + 31 - __clz(static_cast<int>(b2));
    if (b1) return 32 + 31 - __clz(static_cast<int>(b1));
    if (b0) return 31 - __clz(static_cast<int>(b0));
    return -1;
  };
  const bool neg = d66 < 0;
  int top;
  if (!neg) {
    top = top_of(__ballot_sync(FULL, v[0] != 0), __ballot_sync(FULL, v[1] != 0),
                 __ballot_sync(FULL, lane < 3 && v[2] != 0));
  } else if (d66 <= -2) {
    top = kChunks - 1;
  } else {  // d66 == -1: fold into the highest digit below that is not all ones
    const long long FF = 0xFFFFFFFFll;
    top = top_of(__ballot_sync(FULL, v[0] != FF), __ballot_sync(FULL, v[1] != FF),
                 __ballot_sync(FULL, lane < 2 && v[2] != FF));
    if (top < 0) top = 0;
  }
  // canonical chunks: digits below top, the (signed) top, zeros above
  long long ch[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int idx = 32 * r + lane;
    ch[r] = idx < top ? v[r] : idx > top ? 0 : (neg && top < kChunks - 1 ? v[r] - (1ll << 32) : v[r]);
  }
  // 3. magnitude digits m_i (index 0..67; 67 only for the -2^32 top borrow)
  unsigned m[3];
  int h = -1;
  unsigned long long sticky_mask_lo[3];
  if (top >= 0) {
    unsigned z = 0;  // lowest index with a nonzero low word D_i (neg only); top+1 if none
    if (neg) {
      const unsigned n0 = __ballot_sync(FULL, static_cast<unsigned>(ch[0]) != 0u),
                     n1 = __ballot_sync(FULL, static_cast<unsigned>(ch[1]) != 0u),
                     n2 = __ballot_sync(FULL, lane < 3 && static_cast<unsigned>(ch[2]) != 0u);
      z = n0 ? __ffs(n0) - 1 : n1 ? 32 + __ffs(n1) - 1 : n2 ? 64 + __ffs(n2) - 1 : top + 1;
      if (z > static_cast<unsigned>(top)) z = top + 1;
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int idx = 32 * r + lane;
      const unsigned dlo = static_cast<unsigned>(ch[r]);
      if (!neg) {
        m[r] = idx <= top ? dlo : 0u;
      } else if (idx > top + 1 || idx < static_cast<int>(z)) {
        m[r] = 0u;
      } else if (idx == top + 1) {
        m[r] = (z > static_cast<unsigned>(top)) ? 1u : 0u;  // only for an all-zero tail below -2^32
      } else if (idx == static_cast<int>(z)) {
        m[r] = 0u - dlo;
      } else {
        m[r] = ~dlo;
      }
    }
    const unsigned b0 = __ballot_sync(FULL, m[0] != 0), b1 = __ballot_sync(FULL, m[1] != 0),
                   b2 = __ballot_sync(FULL, lane < 4 && m[2] != 0);
    h = top_of(b0, b1, b2);
    sticky_mask_lo[0] = b0;
    sticky_mask_lo[1] = b1;
    sticky_mask_lo[2] = b2;
  }
  // gather the 3-digit window m[h-2..h] to lane 0
  auto digit = [&](int i) -> unsigned {  // collective: all lanes call with the same i
    const int r = i >= 0 ? i >> 5 : 0;
    const unsigned val = r == 0 ? m[0] : r == 1 ? m[1] : m[2];
    const unsigned got = __shfl_sync(FULL, val, i >= 0 ? (i & 31) : 0);
    return i >= 0 ? got : 0u;
  };
  unsigned w0 = 0, w1 = 0, w2 = 0;
  bool sticky = false;
  if (h >= 0) {
    w2 = digit(h);
    w1 = digit(h - 1);
    w0 = digit(h - 2);
    // any nonzero magnitude digit strictly below h - 2
    const int lim = h - 2;
    if (lim > 0) {
      const unsigned long long all_lo =
          sticky_mask_lo[0] | (sticky_mask_lo[1] << 32);  // digits 0..63
      const unsigned long long below =
          lim >= 64 ? all_lo : (all_lo & ((1ull << lim) - 1ull));
      sticky = below != 0ull || (lim > 64 && (sticky_mask_lo[2] & ((1u << (lim - 64)) - 1u)));
    }
  }
  uint64_t ib, nb;
  exsum_resolve_specials(P, M, N, payload, &ib, &nb);
  if (lane == 0 && result) {
    uint64_t bits;
    if (nb) {
      bits = nb;
    } else if (ib) {
      bits = ib;
    } else if (top < 0) {
      bits = 0;
    } else {
      const uint32_t win[3] = {w0, w1, w2};
      const int base = h - 2;  // digit index of win[0] (may be negative: then win[0..] padded)
      bits = exsum_round_digits(win, 3, neg, -1075 + 32 * base, sticky);
    }
    *result = __longlong_as_double(static_cast<long long>(bits));
  }
  if (partial) {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int idx = 32 * r + lane;
      if (idx < kChunks) partial->acc.chunk[idx] = ch[r];
    }
    if (lane == 0) {
      partial->acc.inf_bits = ib;
      partial->acc.nan_bits = nb;
      partial->acc.adds_until_propagate = kCarryTerms;
      partial->acc.reserved_ = 0;
      partial->first_pos_inf = P;
      partial->first_neg_inf = M;
      partial->first_nan = N;
      partial->nan_payload = payload;
    }
  }
}

// --------------------------------------------------------------- K1 + K2 + K3

__global__ void __launch_bounds__(kThreads, 1)
exsum_sum_kernel(const double *__restrict__ x, unsigned long long n,
                 unsigned long long base_index, Workspace *__restrict__ ws, int finalize,
                 double *result, exsum_partial *partial) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_last;
  __shared__ unsigned long long s_spec[4];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char *wsm = smem + warp * kWarpSmem;
  long long *scratch = reinterpret_cast<long long *>(smem + kWarps * kWarpSmem);
  // Programmatic dependent launch: let the next sum in the stream start its CTAs
  // on SMs this grid releases (no-op unless launched with EXSUM_SUM_OVERLAP).
  asm volatile("griddepcontrol.launch_dependents;");
  // K1: contiguous per-warp ranges, boundaries on 4-term multiples.
  const unsigned long long gw = static_cast<unsigned long long>(blockIdx.x) * kWarps + warp;
  const unsigned long long nw = static_cast<unsigned long long>(gridDim.x) * kWarps;
  const unsigned long long quads = (n + 3) >> 2;
  const unsigned long long qb = quads * gw / nw, qe = quads * (gw + 1) / nw;
  const unsigned long long tb = qb * 4, te = min(qe * 4, n);
  if (lane == 0 && te > tb) {  // start the first batches' DRAM reads before zeroing smem
    const uintptr_t p0 = reinterpret_cast<uintptr_t>(x + tb) & ~uintptr_t{15};
    const uintptr_t p1 = reinterpret_cast<uintptr_t>(x + min(te, tb + 2ull * kBatchTerms * 32));
    const uint32_t bytes = static_cast<uint32_t>((p1 - p0 + 15) & ~uintptr_t{15});
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0), "r"(bytes) : "memory");
  }
  zero_warp(wsm, lane);
  __syncwarp();
  const Lane a = acc::lane_view(wsm, lane);
  Specials sp{~0ull, ~0ull, ~0ull};
  int norm_count = 0;
  warp_accumulate(x, tb, te, base_index, a, sp, norm_count, lane);

  // K2: the warp's 67 chunk sums.
  acc::warp_chunks(wsm, a, lane, scratch + warp * kChunks);
  const unsigned long long P = warp_min_u64(sp.P), M = warp_min_u64(sp.M),
                           N = warp_min_u64(sp.N);
  // The workspace is shared with the previous sum in the stream: wait for that
  // grid (complete, memory flushed) before the first workspace access.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (lane == 0) {
    if (P != ~0ull) atomicMax(&ws->inv_pinf, ~P);
    if (M != ~0ull) atomicMax(&ws->inv_ninf, ~M);
    if (N != ~0ull) atomicMax(&ws->inv_nan, ~N);
  }
  __syncthreads();
  // K3: CTA combine -> 67 REDG.ADD.64 into the workspace.
  if (threadIdx.x < kChunks) {
    long long s = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += scratch[w * kChunks + threadIdx.x];
    if (s) atomicAdd(&ws->chunk[threadIdx.x], static_cast<unsigned long long>(s));
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&ws->done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  // Last CTA: gather the workspace in parallel, then one thread rounds.
  __threadfence();
  if (threadIdx.x < kChunks) {
    scratch[threadIdx.x] = static_cast<long long>(__ldcg(&ws->chunk[threadIdx.x]));
    if (finalize) ws->chunk[threadIdx.x] = 0;
  } else if (threadIdx.x < kChunks + 4) {
    const int j = threadIdx.x - kChunks;
    const unsigned long long *src = &ws->inv_pinf;
    s_spec[j] = __ldcg(src + j);  // inv_pinf, inv_ninf, inv_nan, nan_payload
    if (finalize) const_cast<unsigned long long *>(src)[j] = 0;
  }
  __syncthreads();
  if (warp != 0) return;
  const unsigned long long Nf = ~s_spec[2];
  unsigned long long payload = s_spec[3];
  if (Nf != ~0ull && Nf >= base_index && Nf - base_index < n) {
    payload = __ldcg(reinterpret_cast<const unsigned long long *>(x) + (Nf - base_index));
    if (!finalize && lane == 0) ws->nan_payload = payload;  // first NaN so far is in this launch
  }
  if (lane == 0) ws->done = 0;
  if (!finalize) return;
  warp_emit(scratch, ~s_spec[0], ~s_spec[1], Nf, payload, result, partial, lane);
}

// Finalise a workspace filled by exsum_cuda_accumulate launches.
__global__ void exsum_finalize_kernel(Workspace *ws, double *result, exsum_partial *partial) {
  __shared__ long long sc[kChunks];
  if (threadIdx.x < kChunks) {
    sc[threadIdx.x] = static_cast<long long>(ws->chunk[threadIdx.x]);
    ws->chunk[threadIdx.x] = 0;
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const unsigned long long P = ~ws->inv_pinf, M = ~ws->inv_ninf, N = ~ws->inv_nan;
  const unsigned long long payload = ws->nan_payload;
  __syncwarp();
  if (threadIdx.x == 0) {
    ws->inv_pinf = ws->inv_ninf = ws->inv_nan = 0;
    ws->nan_payload = 0;
    ws->done = 0;
  }
  warp_emit(sc, P, M, N, payload, result, partial, threadIdx.x);
}

// ------------------------------------------------------------------------- K4

__global__ void __launch_bounds__(kThreads, 1)
exsum_segmented_kernel(const double *__restrict__ x, const unsigned long long *__restrict__ offs,
                       unsigned long long nseg, Workspace *__restrict__ ws, double *out,
                       exsum_partial *partials) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char *wsm = smem + warp * kWarpSmem;
  long long *row = reinterpret_cast<long long *>(smem + kWarps * kWarpSmem) + warp * kChunks;
  const Lane a = acc::lane_view(wsm, lane);
  while (true) {
    unsigned int s = 0;
    if (lane == 0) s = atomicAdd(&ws->seg_next, 1u);
    s = __shfl_sync(0xffffffffu, s, 0);
    if (s >= nseg) break;
    zero_warp(wsm, lane);
    __syncwarp();
    const unsigned long long b = offs[s], e = offs[s + 1];
    Specials sp{~0ull, ~0ull, ~0ull};
    int norm_count = 0;
    // indices local to the segment: position - b
    warp_accumulate(x, b, e, 0ull - b, a, sp, norm_count, lane);
    acc::warp_chunks(wsm, a, lane, row);
    const unsigned long long P = warp_min_u64(sp.P), M = warp_min_u64(sp.M),
                             N = warp_min_u64(sp.N);
    __syncwarp();
    const unsigned long long payload =
        N != ~0ull ? __ldg(reinterpret_cast<const unsigned long long *>(x) + b + N) : 0ull;
    warp_emit(row, P, M, N, payload, out + s, partials ? partials + s : nullptr, lane);
    __syncwarp();
  }
  // Last warp out resets the claim counters for the next launch.
  if (lane == 0) {
    const unsigned int total = gridDim.x * kWarps;
    if (atomicAdd(&ws->seg_done, 1u) == total - 1) {
      ws->seg_next = 0;
      ws->seg_done = 0;
    }
  }
}

// ------------------------------------------------------------------------- K5

__global__ void exsum_merge_kernel(const exsum_partial *parts, unsigned long long k,
                                   double *result, exsum_partial *out) {
  __shared__ long long sc[kChunks];
  __shared__ unsigned long long sP, sM, sN, sPay;
  const int t = threadIdx.x;
  if (t < kChunks) {
    long long s = 0;
    for (unsigned long long j = 0; j < k; ++j) s += parts[j].acc.chunk[t];
    sc[t] = s;
  }
  if (t == 0) {
    unsigned long long P = ~0ull, M = ~0ull, N = ~0ull, pay = 0;
    for (unsigned long long j = 0; j < k; ++j) {
      P = min(P, static_cast<unsigned long long>(parts[j].first_pos_inf));
      M = min(M, static_cast<unsigned long long>(parts[j].first_neg_inf));
      if (parts[j].first_nan < N) {
        N = parts[j].first_nan;
        pay = parts[j].nan_payload;
      }
    }
    sP = P;
    sM = M;
    sN = N;
    sPay = pay;
  }
  __syncthreads();
  if (t < 32) warp_emit(sc, sP, sM, sN, sPay, result, out, t);
}

}  // namespace dev
}  // namespace exsum_b200

// ===================================================================== C ABI

using namespace exsum_b200;
using namespace exsum_b200::dev;

namespace {

constexpr int kMaxDevices = 64;
int g_num_sms[kMaxDevices] = {};
bool g_configured[kMaxDevices] = {};

// Per-device one-time setup: SM count and the >48 KB dynamic smem opt-in.
int prepare_device(int *sms) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return EXSUM_ECUDA;
  if (!g_configured[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      return EXSUM_ECUDA;
    if (cudaFuncSetAttribute(exsum_sum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmem) != cudaSuccess ||
        cudaFuncSetAttribute(exsum_segmented_kernel,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) != cudaSuccess)
      return EXSUM_ECUDA;
    g_num_sms[dev] = n;
    g_configured[dev] = true;
  }
  *sms = g_num_sms[dev];
  return EXSUM_OK;
}

int launch_status() { return cudaGetLastError() == cudaSuccess ? EXSUM_OK : EXSUM_ECUDA; }

// Grid for a sum of n terms: one CTA per SM, fewer for small inputs (keep at
// least ~4 K terms per warp so the per-CTA fixed cost stays amortised).
unsigned grid_for(unsigned long long n, int sms) {
  const unsigned long long per_cta = 4096ull * kWarps;
  unsigned long long g = (n + per_cta - 1) / per_cta;
  if (g < 1) g = 1;
  if (g > static_cast<unsigned long long>(sms)) g = sms;
  return static_cast<unsigned>(g);
}

int sum_launch(const double *d_x, size_t n, uint64_t base_index, void *d_ws, size_t ws_bytes,
               void *stream, int finalize, double *d_result, exsum_partial *d_partial,
               unsigned flags = 0) {
  if (!d_ws || ws_bytes < sizeof(Workspace) || (n && !d_x)) return EXSUM_EINVAL;
  int sms = 0;
  const int st = prepare_device(&sms);
  if (st) return st;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid_for(n, sms));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  if (flags & EXSUM_SUM_OVERLAP) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  if (cudaLaunchKernelEx(&cfg, exsum_sum_kernel, d_x, static_cast<unsigned long long>(n),
                         static_cast<unsigned long long>(base_index),
                         static_cast<Workspace *>(d_ws), finalize, d_result, d_partial) !=
      cudaSuccess)
    return EXSUM_ECUDA;
  return launch_status();
}

}  // namespace

extern "C" {

size_t exsum_cuda_workspace_bytes(void) { return sizeof(Workspace); }

int exsum_cuda_workspace_init(void *d_ws, size_t ws_bytes, void *stream) {
  if (!d_ws || ws_bytes < sizeof(Workspace)) return EXSUM_EINVAL;
  return cudaMemsetAsync(d_ws, 0, sizeof(Workspace), static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess
             ? EXSUM_OK
             : EXSUM_ECUDA;
}

int exsum_cuda_sum(const double *d_x, size_t n, uint64_t base_index, double *d_result,
                   exsum_partial *d_partial, void *d_ws, size_t ws_bytes, void *stream) {
  return sum_launch(d_x, n, base_index, d_ws, ws_bytes, stream, 1, d_result, d_partial);
}

int exsum_cuda_sum_ex(const double *d_x, size_t n, uint64_t base_index, double *d_result,
                      exsum_partial *d_partial, void *d_ws, size_t ws_bytes, void *stream,
                      unsigned flags) {
  return sum_launch(d_x, n, base_index, d_ws, ws_bytes, stream, 1, d_result, d_partial, flags);
}

int exsum_cuda_accumulate(const double *d_x, size_t n, uint64_t base_index, void *d_ws,
                          size_t ws_bytes, void *stream) {
  if (n == 0) return (d_ws && ws_bytes >= sizeof(Workspace)) ? EXSUM_OK : EXSUM_EINVAL;
  return sum_launch(d_x, n, base_index, d_ws, ws_bytes, stream, 0, nullptr, nullptr);
}

int exsum_cuda_finalize(double *d_result, exsum_partial *d_partial, void *d_ws, size_t ws_bytes,
                        void *stream) {
  if (!d_ws || ws_bytes < sizeof(Workspace)) return EXSUM_EINVAL;
  exsum_finalize_kernel<<<1, 96, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<Workspace *>(d_ws), d_result, d_partial);
  return launch_status();
}

int exsum_cuda_sum_segmented(const double *d_x, const uint64_t *d_offsets, size_t nseg,
                             double *d_out, exsum_partial *d_partials, void *d_ws,
                             size_t ws_bytes, void *stream) {
  if (!d_ws || ws_bytes < sizeof(Workspace) || (nseg && (!d_offsets || !d_out)))
    return EXSUM_EINVAL;
  if (nseg == 0) return EXSUM_OK;
  if (nseg >= 0xFFFFFFFFull) return EXSUM_EINVAL;
  int sms = 0;
  const int st = prepare_device(&sms);
  if (st) return st;
  unsigned long long g = (nseg + kWarps - 1) / kWarps;
  if (g > static_cast<unsigned long long>(sms)) g = sms;
  exsum_segmented_kernel<<<static_cast<unsigned>(g), kThreads, kSmem,
                           static_cast<cudaStream_t>(stream)>>>(
      d_x, reinterpret_cast<const unsigned long long *>(d_offsets), nseg,
      static_cast<Workspace *>(d_ws), d_out, d_partials);
  return launch_status();
}

int exsum_cuda_merge(const exsum_partial *d_parts, size_t k, double *d_result,
                     exsum_partial *d_out, void *stream) {
  if (k && !d_parts) return EXSUM_EINVAL;
  exsum_merge_kernel<<<1, 96, 0, static_cast<cudaStream_t>(stream)>>>(d_parts, k, d_result,
                                                                      d_out);
  return launch_status();
}

}  // extern "C"
