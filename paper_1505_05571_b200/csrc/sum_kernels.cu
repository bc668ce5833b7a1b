// sum_kernels.cu — the sm_100a exact-summation hot path.
//
// Replaces exact_sum(values, ExactMethod::large) (vector_ops.cpp:121-130), i.e.
// LargeAccumulator::add(span) + drain + SmallAccumulator::round
// (large_accumulator.cpp:28-136, small_accumulator.cpp:244-348), and the
// split-merge of parallel_exact_sum (vector_ops.cpp:172-186).  See DESIGN.md.
//
// Device representation (B200-first, not the reference's): every LANE owns a
// private fixed-point superaccumulator in shared memory, so a term costs one
// conflict-free read-modify-write, no atomics, independent of the exponent
// distribution.  Two layouts:
//   EXSUM_RIPPLE = 1 (default, round 2): two unsigned planes (positive and
//     negative terms) of 67 32-bit words, word r of weight 2^(32 r - 1075) (the
//     reference's chunk weight): 536 B per lane, 12 warps per SM.  A term
//     (-1)^s m 2^(e' - 1075), e' = max(e, 1), adds m << (e' & 31) (three words)
//     at word e' >> 5 of plane s; the rare carry out of the third word ripples
//     upward at once, so there is no carry budget and no renormalisation.
//   EXSUM_RIPPLE = 0 (round 1): 66 slots, slot k a signed 96-bit integer of
//     weight 2^(32k - 1075) stored as a u32 plane L[k][lane] and an s64 plane
//     H[k][lane] (25.3 KB per warp, 8 warps per SM); 2^11 of headroom per slot
//     = 2047 terms, each lane renormalises at most every 2016 terms.
// The kernels are latency-bound on the shared read-modify-write chain, so warps
// per SM are the lever: 8 -> 12 warps took config 3 from 5.84 to 6.34 TB/s and
// config 5 from 5.44 to 6.09 TB/s at the same ~23.5 instructions per term
// (profiles/r02_ripple_ab.log, r02_ripple_knobs.log: 10 warps 5.76 / 5.63).
//
// Why not the reference's 4096 shared bins: 64-bit shared atomics compile to
// ATOMS.CAST.SPIN.64 CAS loops on sm_100a, random-bin read-modify-writes cost
// ~3.5x in bank conflicts, and U[0,1) puts half of all terms in one bin; even
// without counts or transfers that step measures 0.04-2.0 TB/s
// (scripts/probes/bins.cu, profiles/r01_probe_bins.log).
//
// Per-term cost: ~23.5 SASS instructions (13 integer ALU, 4 FMA-pipe IMADs, 6
// LSU) and 6 shared wavefronts.  Loads are 256-bit (LDG.E.EF.ENL2.256),
// "rolling": a vector's registers are refilled with the next batch's vector
// right after its four terms are added, with one 8 KB cp.async.bulk L2
// prefetch per warp one batch further ahead (predicated on lane 0: no branch).  When every lane's batch falls in one slot (narrow
// exponent ranges) the batch is summed in registers and the slot gets one
// read-modify-write; when each lane's batch also has one sign (U[0,1)), the
// magnitudes are summed without the sign complement (8.5 instructions/term).
// A warp whose first batch is not one-slot runs a loop compiled without that
// fast path (EXSUM_UNIFORM_DISPATCH).  Inf/NaN are added blindly and cancelled
// by a per-batch fix-up (pipelined one batch behind in the segmented kernel,
// EXSUM_SEG_FIX_GROUP).  Sustained
// rates sit at the 1 kW power cap, so energy per term (not DRAM) bounds the
// general path.
//
// Term sources (kOp): x[i]; fl(x[i]^2) for sqnorm; fl(a[i] b[i]) for dot, with
// the reference's x86 NaN rules applied in the fix-up.
//
// Kernels
//   exsum_sum_kernel<kOp>   K1+K2+K3: persistent grid (1 CTA per SM; 8/9 of the
//                           SMs for short overlapped sums), each warp streams a
//                           contiguous range; the CTA combines its lanes into 67
//                           chunk sums, REDG.ADD.64 into the workspace; the last
//                           CTA canonicalises, resolves Inf/NaN by first index
//                           and rounds (warp-parallel).  Launchable with
//                           programmatic dependent launch.  With P2P arguments
//                           the last CTA also exchanges the record with the
//                           other ranks over peer memory and merges
//                           (exsum_p2p_sum); with a group split, one cooperative
//                           launch emulates several ranks (tests).
//   exsum_wsum_kernel       K1w: the windowed first phase of plain sums of
//                           >= 2^28 terms (16 warps per SM, a 16-slot window per
//                           warp); exsum_sum_kernel then sums what it left
//                           ("jobs") or returns at once if it left nothing.
//   exsum_segmented_kernel  K4: one warp per segment (dynamic claim), compact
//                           loop body (instruction-cache bound otherwise).
//   exsum_merge_kernel      K5: merge of k gathered partial records + round.
//   exsum_finalize_kernel   round a workspace filled by incremental launches.

#include <cuda_runtime.h>
#include <stdint.h>

#include <string.h>

#include <atomic>
#include <mutex>
#include <type_traits>

#include "exsum_b200.h"
#include "exsum_core.h"
#include "exsum_nvtx.h"

#ifndef EXSUM_RIPPLE
#define EXSUM_RIPPLE 1  // lane accumulators as two unsigned planes of 32-bit words with immediate
                        // carry ripple (536 B per lane, 12 warps per SM) instead of 66 signed
                        // 96-bit slots with deferred carries (792 B per lane, 8 warps per SM)
#endif
#ifndef EXSUM_VEC_PER_LANE
#define EXSUM_VEC_PER_LANE 8  // single-sum kernel: 256-bit vectors per lane per batch
#endif
#ifndef EXSUM_SQNORM_VEC
#define EXSUM_SQNORM_VEC 4  // sqnorm kernel: vectors per lane per batch (1e8 U[-1,1): 6130 GB/s; 3: 6214,
                            // 5: 5811, 8: 4823 — a smaller loop body at 12 warps; r02_products_vec.log)
#endif
#ifndef EXSUM_DOT_VEC
#define EXSUM_DOT_VEC 2  // dot kernel: vectors per lane per batch (x and y each; 2: 6751 / 6640 GB/s
                         // co-aligned / misaligned, 3: 6697 / 6524, 4: 6592 / 6287; r02_products_vec.log)
#endif
#ifndef EXSUM_SEG_VEC
#define EXSUM_SEG_VEC 7  // segmented kernel: vectors per lane per batch (7: config 5 2.083 -> 2.068 ms
                         // vs 8, a smaller loop body; 6: 2.105; r02_knob_resweep_seg.log)
#endif
#ifndef EXSUM_PREFETCH_BATCHES
#define EXSUM_PREFETCH_BATCHES 1  // L2 bulk-prefetch distance, in batches
#endif
#ifndef EXSUM_UNIFORM_FAST
#define EXSUM_UNIFORM_FAST 1  // single-sum kernel: register fast path for one-slot batches
#endif
#ifndef EXSUM_INTERLEAVE
#define EXSUM_INTERLEAVE 1  // single sums: batches round-robin over warps (1) instead of
                           // contiguous per-warp ranges (0): all warps sweep one window
#endif
#ifndef EXSUM_SEG_AHEAD
#define EXSUM_SEG_AHEAD 0  // segmented: claim the next segment at the start of the current one and
                           // prefetch its head into L2 before the current epilogue
#endif
#ifndef EXSUM_SEG_PF_NEXT
#define EXSUM_SEG_PF_NEXT 0  // segmented: L2 prefetch of the next (already claimed) segment's head
                             // right after the current segment's chunk sums
#endif
#ifndef EXSUM_SEG_SPLIT
#define EXSUM_SEG_SPLIT EXSUM_RIPPLE  // segmented kernel: unguarded full batches + a one-vector tail
                                     // loop (config 5: +1.1% with the ripple accumulators, r02_ripple_knobs.log;
                                     // no gain with the slot accumulators, r02_variants_segsplit.log)
#endif
#ifndef EXSUM_FP64_DECODE
#define EXSUM_FP64_DECODE 0  // general path: slot value by FP64 scaling + conversions (idle FP64
                             // and conversion pipes) instead of the integer decode
#endif
#ifndef EXSUM_XOR_LOP
#define EXSUM_XOR_LOP 1  // sign complement with two LOP3 (ALU) instead of LEA + 2 IMAD (FMA)
#endif
#ifndef EXSUM_TIMELINE
#define EXSUM_TIMELINE 0  // diagnostics build: per-warp %globaltimer stamps (scripts/timeline.py)
#endif
#ifndef EXSUM_FIX_L1
#define EXSUM_FIX_L1 2  // scanning Inf/NaN fix-up re-reads: 0 ld.global.cg of each high word (L2
                        // round trips), 1 the same L1-allocating (the batch's lines are often still
                        // in L1; the flagged term's full re-read hits the scanned sector), 2 whole
                        // 32-byte vectors, L1-allocating (8 wavefronts per 4 terms instead of per
                        // term).  Config 5: 2.255 / 2.196 / 2.176 ms; 2-4 neutral
                        // (r01_variants_fixup.log)
#endif
#ifndef EXSUM_UNIFORM_SIGNED
#define EXSUM_UNIFORM_SIGNED 1  // one-slot batches (slot >= 1) whose lanes each hold one sign: sum
                                // the magnitudes (no sign complement, no denormal handling; 8
                                // instructions per term instead of ~16), negate once per lane
#endif
#ifndef EXSUM_PF_ALIGNED
#define EXSUM_PF_ALIGNED 1  // L2 prefetch of the (32-byte aligned) x stream without the 16-byte
                            // rounding arithmetic
#endif
#ifndef EXSUM_PF_PRED
#define EXSUM_PF_PRED 1  // plain sums: the per-batch L2 prefetch predicated on lane 0 instead of a
                         // lane-0 branch
#endif
#ifndef EXSUM_SEG_DEFER
#define EXSUM_SEG_DEFER 1  // segmented sums: round every segment in a second launch
                           // (exsum_segment_emit_kernel) instead of on the streaming warp
#endif
#ifndef EXSUM_SEG_FIX_GROUP
#define EXSUM_SEG_FIX_GROUP 1  // segmented sums: pipelined Inf/NaN fix-up, flags per group of this
                               // many vectors (0: the synchronous scanning fix-up); config 5:
                               // 2.087 / 2.095 / 2.108 ms for 1 / 2 / 0 (r02_segfix.log)
#endif
#ifndef EXSUM_DEBUG_CHECKS
#define EXSUM_DEBUG_CHECKS 0  // debug build: every streaming load checks its vector index against
                              // the range end (printf + trap on a violation)
#endif
#if EXSUM_DEBUG_CHECKS
#include <cstdio>
#define EXSUM_DCHECK(c)                                                          \
  do {                                                                           \
    if (!(c)) {                                                                  \
      printf("EXSUM_DCHECK failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);       \
      __trap();                                                                  \
    }                                                                            \
  } while (0)
#else
#define EXSUM_DCHECK(c) \
  do {                  \
  } while (0)
#endif
#ifndef EXSUM_LDG_KIND
#define EXSUM_LDG_KIND 2  // 256-bit loads: 0 nc+L1::no_allocate, 1 nc, 2 nc+L1::evict_first (3-4%
                          // faster on configs 3-5 than 0: r01_variants_ldg.log), 3 plain
#endif
#ifndef EXSUM_SUM_SCAN
#define EXSUM_SUM_SCAN 1  // single-sum kernel: scanning Inf/NaN fix-up (0: per-term loop; 1.43x
                          // faster on 1e-4 Inf/NaN data, neutral otherwise: r01_variants_sumscan.log)
#endif
#ifndef EXSUM_UNIFORM_DISPATCH
#define EXSUM_UNIFORM_DISPATCH 1  // one-slot fast path: a warp whose first batch is not one-slot runs a
                                  // loop without the fast path's code (kept only for warps that start
                                  // one-slot; it still backs off per batch there)
#endif
#ifndef EXSUM_UNIFORM_BACKOFF
#define EXSUM_UNIFORM_BACKOFF 7  // batches to skip the one-slot test after a miss
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
  unsigned int wdone;     // two-phase: windowed CTAs finished (zero between calls)
};

struct Specials {                // first occurrences seen by one lane
  unsigned long long P, M, N;    // index (global or segment-local), ~0 = none
};

__device__ __forceinline__ uint32_t exponent_field(uint32_t hi) { return (hi >> 20) & 0x7FFu; }

// ------------------------------------------------------ lane accumulators

#ifndef EXSUM_WARPS
#define EXSUM_WARPS (EXSUM_RIPPLE ? 12 : 8)  // warps per CTA (one CTA per SM)
#endif
#ifndef EXSUM_SLOTS
#define EXSUM_SLOTS 66  // 65: one carry-only slot (fits a 9th warp in shared memory)
#endif
constexpr int kWarps = EXSUM_WARPS;
constexpr int kThreads = kWarps * 32;
constexpr int kSlots = EXSUM_SLOTS;  // slots 0..63 take terms (e' >> 5), the rest only carries
static_assert(kSlots == 65 || kSlots == 66, "slot count");
constexpr int kLPlane = kSlots * 32 * 4;
constexpr int kHPlane = kSlots * 32 * 8;
#if EXSUM_RIPPLE
// Two warps share a region of kChunks rows of 512 B: row r = word r (weight
// 2^(32 r - 1075)) of four planes, [warp & 1][sign][lane] x 4 B.
static_assert(kWarps % 2 == 0, "warps pair up");
constexpr int kRowBytes = 512;
constexpr int kPairSmem = kChunks * kRowBytes;          // 34,304 B
constexpr int kAccSmem = (kWarps / 2) * kPairSmem;      // 205,824 B (12 warps)
#else
constexpr int kWarpSmem = kLPlane + kHPlane;            // 25,344 B
constexpr int kAccSmem = kWarps * kWarpSmem;
#endif
constexpr int kScratch = kWarps * kChunks * 8;          // per-warp chunk rows
constexpr int kSmem = kAccSmem + kScratch;              // 207,040 B (8 warps, 66 slots)
constexpr int kPrefetchBatches = EXSUM_PREFETCH_BATCHES;
constexpr int kUniformBackoff = EXSUM_UNIFORM_BACKOFF;

#if EXSUM_TIMELINE
// [warp][0..3]: start, loop end, flush end (after the CTA's REDs), last-CTA end
__device__ unsigned long long g_timeline[148 * 16 * 4 + 8];
// segmented kernel: per warp, summed phase durations (ns) over its segments:
// [0] claim, [1] clear, [2] accumulate, [3] chunks, [4] emit, [5] segments, [6] terms
__device__ unsigned long long g_seg_timeline[148 * 16 * 8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define EXSUM_STAMP(slot)                                                                  \
  do {                                                                                     \
    if (lane == 0 && blockIdx.x < 148)                                                     \
      g_timeline[(blockIdx.x * kWarps + warp) * 4 + (slot)] = gtimer();                    \
  } while (0)
#else
#define EXSUM_STAMP(slot) \
  do {                    \
  } while (0)
#endif
static_assert(kSmem <= 227 * 1024, "shared memory budget");

// One lane's view of its accumulator.  Generic pointers serve the cold paths;
// the hot path uses 32-bit shared addresses: slot k's low word at sl + 128 k,
// its high word at 2 (sl + 128 k) + hoff.
struct Lane {
  uint32_t *L;            // &Lplane[0][lane]; slot k at L[32 k]
  unsigned long long *H;  // &Hplane[0][lane]; slot k at H[32 k]
  uint32_t sl;
  uint32_t hoff;
  uint32_t two;   // 2 and 128, opaque to ptxas: keeps the address arithmetic
  uint32_t c128;  // IMADs on the FMA pipe instead of LEAs on the ALU pipe
  uint32_t one;   // EXSUM_RIPPLE: 1, opaque likewise (L: word 0 of the positive plane,
                  // word r at L[128 r], the negative plane 32 words above; H unused)
};

#if EXSUM_RIPPLE
__device__ __forceinline__ unsigned char *warp_base(unsigned char *smem, int warp) {
  return smem + (warp >> 1) * kPairSmem + (warp & 1) * 256;
}

__device__ __forceinline__ Lane lane_view(unsigned char *warp_smem, int lane) {
  Lane v;
  v.L = reinterpret_cast<uint32_t *>(warp_smem) + lane;
  v.H = nullptr;
  v.sl = static_cast<uint32_t>(__cvta_generic_to_shared(v.L));
  v.hoff = 0u;
  v.one = (blockDim.x >> 30) + 1u;
  v.two = v.one + v.one;
  v.c128 = v.two * 64u;
  return v;
}

// Zero one warp's two planes: 256 contiguous bytes in each of the 67 rows.
__device__ __forceinline__ void zero_warp(unsigned char *warp_smem, int lane) {
#pragma unroll 8
  for (int r = 0; r < kChunks; ++r)
    *reinterpret_cast<uint2 *>(warp_smem + r * kRowBytes + lane * 8) = make_uint2(0u, 0u);
}
#else
__device__ __forceinline__ unsigned char *warp_base(unsigned char *smem, int warp) {
  return smem + warp * kWarpSmem;
}

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

// Zero one warp's accumulator cooperatively with 16-byte stores.
__device__ __forceinline__ void zero_warp(unsigned char *warp_smem, int lane) {
  uint4 *p = reinterpret_cast<uint4 *>(warp_smem);
  constexpr int n16 = kWarpSmem / 16;
#pragma unroll 4
  for (int i = lane; i < n16; i += 32) p[i] = make_uint4(0, 0, 0, 0);
}


#endif

// The term as three 32-bit words of its complemented, shifted significand
// (u2:u1:u0 = s ? ~(m << sh) : m << sh; a negative term's +1 is the carry-in
// s + s) and e' = max(e, 1).  The B200 integer ALU pipe and the FMA pipe each
// retire 16 lanes/clk/SMSP (measured, profiles/r01_pipe_probe_*); the decode
// keeps a few IMADs on the FMA pipe, but the sign complement is two LOP3s: one
// instruction fewer per term than IMAD-based xor (x (2s + 1) + s), which
// measured faster both in bursts and under the power cap
// (profiles/r01_variants_xorlop.log).
__device__ __forceinline__ void decode96(uint32_t lo, uint32_t hi, uint32_t e, uint32_t &s,
                                         uint32_t &u0, uint32_t &u1, uint32_t &u2,
                                         uint32_t &ep) {
  uint32_t d, mhi, mh, m1, lx, mx;
  asm("shr.s32 %0, %1, 31;" : "=r"(s) : "r"(hi));                         // ALU: sign mask
  asm("max.u32 %0, %1, 1;" : "=r"(ep) : "r"(e));                         // ALU
  asm("mad.lo.u32 %0, %1, -1, %2;" : "=r"(d) : "r"(e), "r"(ep));          // FMA: 1 iff e == 0
  asm("lop3.b32 %0, %1, 0xFFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x100000u));  // (a&b)|c
  asm("mad.lo.u32 %0, %1, -1048576, %2;" : "=r"(mh) : "r"(d), "r"(mhi));  // FMA: drop implicit 1
#if EXSUM_XOR_LOP
  (void)m1;
  asm("xor.b32 %0, %1, %2;" : "=r"(lx) : "r"(lo), "r"(s));                 // ALU: lo ^ s
  asm("xor.b32 %0, %1, %2;" : "=r"(mx) : "r"(mh), "r"(s));                 // ALU: mh ^ s
#else
  asm("mad.lo.u32 %0, %1, 2, 1;" : "=r"(m1) : "r"(s));                    // FMA: +-1
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(lx) : "r"(lo), "r"(m1), "r"(s));  // FMA: lo ^ s
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(mx) : "r"(mh), "r"(m1), "r"(s));  // FMA: mh ^ s
#endif
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u0) : "r"(s), "r"(lx), "r"(ep));   // shift mod 32
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u1) : "r"(lx), "r"(mx), "r"(ep));
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u2) : "r"(mx), "r"(s), "r"(ep));
}

#define EXSUM_RMW_LD "ld.shared.u32 l, [%0];\n\tld.shared.v2.u32 {h0, h1}, [%1];\n\t"
#define EXSUM_RMW_ST "st.shared.u32 [%0], l;\n\tst.shared.v2.u32 [%1], {h0, h1};\n\t}"

#if EXSUM_RIPPLE
// ---- two unsigned planes of 32-bit words, carries rippled at once ----
// A lane's sum is P - N, each plane an unsigned 2144-bit integer in 67 words
// (word r of weight 2^(32 r - 1075): the reference's chunk weight).  A term adds
// its magnitude m << (e' & 31) (three words) to words e' >> 5 .. + 2 of its
// sign's plane; a carry out of the third word (probability ~2^-12 per term) is
// rippled upward right after the vector's four terms.  Planes only grow, so the
// ripple is amortised O(1) for any input (a carry through j all-ones words
// clears them); there is no carry budget and no renormalisation.  The blind
// add of an Inf/NaN term (slot 63: words 63..65, word 66 takes the ripple) is
// cancelled by subtracting the same magnitude from the same plane.

// Shared address of word e >> 5 of the term's plane: PRMT puts the high byte
// (s << 7 | e >> 4) in byte 1 and its replicated sign in byte 0, so one AND
// leaves (e >> 5) << 9 | s << 7 = row * 512 + sign * 128.
__device__ __forceinline__ uint32_t word_addr(const Lane &a, uint32_t hi) {
  uint32_t r, t, la;
  asm("prmt.b32 %0, %1, %2, 0x443B;" : "=r"(r) : "r"(hi), "r"(0u));
  asm("and.b32 %0, %1, 0x7E80;" : "=r"(t) : "r"(r));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(la) : "r"(t), "r"(a.one), "r"(a.sl));
  return la;
}

// u2:u1:u0 = m << (e' & 31), e' = max(e, 1), m without the implicit bit for e = 0.
__device__ __forceinline__ void decode_mag(uint32_t lo, uint32_t hi, uint32_t e, uint32_t &u0,
                                           uint32_t &u1, uint32_t &u2) {
  uint32_t ep, d, mhi, mh;
  asm("max.u32 %0, %1, 1;" : "=r"(ep) : "r"(e));                          // ALU
  asm("mad.lo.u32 %0, %1, -1, %2;" : "=r"(d) : "r"(e), "r"(ep));           // FMA: 1 iff e == 0
  asm("lop3.b32 %0, %1, 0xFFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x100000u));
  asm("mad.lo.u32 %0, %1, -1048576, %2;" : "=r"(mh) : "r"(d), "r"(mhi));   // FMA: drop implicit 1
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u0) : "r"(0u), "r"(lo), "r"(ep));
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u1) : "r"(lo), "r"(mh), "r"(ep));
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u2) : "r"(mh), "r"(0u), "r"(ep));
}

// + 1 at the word at shared address addr, rippling while words wrap to zero.
__device__ __forceinline__ void ripple_up(uint32_t addr) {
  uint32_t w;
#pragma unroll 1
  do {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(addr) : "memory");
    w += 1u;
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(w) : "memory");
    addr += kRowBytes;
  } while (w == 0u);
}

// - 1 likewise (the plane holds at least what is being removed).
__device__ __forceinline__ void ripple_down(uint32_t addr) {
  uint32_t w;
#pragma unroll 1
  do {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(addr) : "memory");
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(w - 1u) : "memory");
    addr += kRowBytes;
  } while (w == 0u);
}

// words [la], [la + 512], [la + 1024] += u0, u1, u2; cb = 2 cb + carry out
__device__ __forceinline__ void words_add(uint32_t la, uint32_t u0, uint32_t u1, uint32_t u2,
                                          uint32_t &cb) {
  asm volatile(
      "{\n\t.reg .u32 w0, w1, w2;\n\t"
      "ld.shared.u32 w0, [%1];\n\t"
      "ld.shared.u32 w1, [%1+512];\n\t"
      "ld.shared.u32 w2, [%1+1024];\n\t"
      "add.cc.u32 w0, w0, %2;\n\t"
      "addc.cc.u32 w1, w1, %3;\n\t"
      "addc.cc.u32 w2, w2, %4;\n\t"
      "addc.u32 %0, %0, %0;\n\t"
      "st.shared.u32 [%1], w0;\n\t"
      "st.shared.u32 [%1+512], w1;\n\t"
      "st.shared.u32 [%1+1024], w2;\n\t}"
      : "+r"(cb)
      : "r"(la), "r"(u0), "r"(u1), "r"(u2)
      : "memory");
}

// One term of a vector: cb collects the carries (bit 3 - q for term q of 4).
__device__ __forceinline__ void add_term_cb(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e,
                                            uint32_t &cb) {
  uint32_t u0, u1, u2;
  decode_mag(lo, hi, e, u0, u1, u2);
  words_add(word_addr(a, hi), u0, u1, u2, cb);
}

// The carries of a vector's four terms (cold).
__device__ __forceinline__ void ripple_fix4(const Lane &a, const uint32_t (&hi)[4], uint32_t cb) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (cb & (8u >> q)) ripple_up(word_addr(a, hi[q]) + 3 * kRowBytes);
}

__device__ __forceinline__ void add_term(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e) {
  uint32_t cb = 0u;
  add_term_cb(a, lo, hi, e, cb);
  if (__builtin_expect(cb != 0u, 0)) ripple_up(word_addr(a, hi) + 3 * kRowBytes);
}

// Remove exactly what add_term added for the term (lo, hi).
__device__ __forceinline__ void cancel_term(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e) {
  uint32_t u0, u1, u2, bw;
  decode_mag(lo, hi, e, u0, u1, u2);
  const uint32_t la = word_addr(a, hi);
  asm volatile(
      "{\n\t.reg .u32 w0, w1, w2;\n\t"
      "ld.shared.u32 w0, [%1];\n\t"
      "ld.shared.u32 w1, [%1+512];\n\t"
      "ld.shared.u32 w2, [%1+1024];\n\t"
      "sub.cc.u32 w0, w0, %2;\n\t"
      "subc.cc.u32 w1, w1, %3;\n\t"
      "subc.cc.u32 w2, w2, %4;\n\t"
      "subc.u32 %0, 0, 0;\n\t"
      "st.shared.u32 [%1], w0;\n\t"
      "st.shared.u32 [%1+512], w1;\n\t"
      "st.shared.u32 [%1+1024], w2;\n\t}"
      : "=r"(bw)
      : "r"(la), "r"(u0), "r"(u1), "r"(u2)
      : "memory");
  if (bw != 0u) ripple_down(la + 3 * kRowBytes);
}

// A signed 96-bit value (a one-slot batch summed in registers) into word k ..
// k + 2 of the plane of its sign.
__device__ __forceinline__ void slot_add96(const Lane &a, uint32_t k, uint32_t v0, uint32_t v1,
                                           uint32_t v2) {
  const uint32_t neg = static_cast<uint32_t>(static_cast<int32_t>(v2) >> 31);
  uint32_t m0 = v0 ^ neg, m1 = v1 ^ neg, m2 = v2 ^ neg;
  asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, 0;\n\taddc.u32 %2, %2, 0;"
      : "+r"(m0), "+r"(m1), "+r"(m2)
      : "r"(neg & 1u));
  const uint32_t la = a.sl + k * kRowBytes + (neg & 128u);
  uint32_t cb = 0u;
  words_add(la, m0, m1, m2, cb);
  if (cb != 0u) ripple_up(la + 3 * kRowBytes);
}

__device__ __forceinline__ void normalize(const Lane &) {}  // nothing is deferred

// The warp's exact sum as 67 chunk values: chunk r = sum over lanes of
// P[r] - N[r] (|chunk| < 2^37).  Lane j sums rows j, j + 32, j + 64 with
// bank-skewed 128-bit reads (the 8 lanes of a wavefront hit 8 bank groups).
__device__ __forceinline__ void warp_chunks(unsigned char *warp_smem, int lane, long long *row) {
  __syncwarp();
#pragma unroll
  for (int rr = 0; rr < 3; ++rr) {
    const int r = 32 * rr + lane;
    if (r < kChunks) {
      const uint4 *p = reinterpret_cast<const uint4 *>(warp_smem + r * kRowBytes);
      long long acc = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int idx = (i + lane) & 15;
        const uint4 v = p[idx];
        const long long t = static_cast<long long>(v.x) + v.y + static_cast<long long>(v.z) + v.w;
        acc += (idx & 8) ? -t : t;
      }
      row[r] = acc;
    }
  }
}
#else
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

// Add one term (exponent field e != 2047, or 2047 for the blind add of an
// Inf/NaN that the batch fix-up cancels) to the lane's slots.
#if EXSUM_FP64_DECODE
// The slot value of x as a signed 96-bit integer h * 2^32 + u0 computed on the
// FP64 and conversion pipes: slot k = e >> 5 (e = 0 and 1 share slot 0), value
// y = x * 2^(1075 - 32k) = s m 2^(e' & 31) — the integer decode's value.
// t = y / 2^32 = (x * 2^(1011 - 32k)) * 2^32: both products exact (x * A_k lies
// in [2^-63, 2^20) for every finite x of slot k, denormals included), then
// h = floor(t) and u0 = (t - h) * 2^32, both exact integers.  An Inf/NaN decodes
// to garbage (saturated / zero conversions) that cancel_term removes exactly.
__device__ __forceinline__ void decode_fp64(uint32_t lo, uint32_t hi, uint32_t e, uint32_t &k,
                                            uint32_t &u0, long long &h) {
  k = e >> 5;
  uint32_t ahi;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(ahi) : "r"(k), "r"(0xFE000000u), "r"(2034u << 20));
  const double A = __hiloint2double(static_cast<int>(ahi), 0);
  const double x = __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
  const double t = __dmul_rn(__dmul_rn(x, A), 4294967296.0);
#if EXSUM_FP64_DECODE == 2
  // low word on the integer pipes: (m << (e' & 31)) mod 2^32, negated for x < 0
  // (the two's complement's low word; h = floor(t) is the matching high part)
  uint32_t ep, w, sg;
  asm("max.u32 %0, %1, 1;" : "=r"(ep) : "r"(e));
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(w) : "r"(0u), "r"(lo), "r"(ep));
  asm("shr.s32 %0, %1, 31;" : "=r"(sg) : "r"(hi));
  u0 = (w ^ sg) - sg;
  h = __double2ll_rd(t);
#else
  const double th = floor(t);
  u0 = __double2uint_rz(__dmul_rn(__dsub_rn(t, th), 4294967296.0));
  h = __double2ll_rz(th);
#endif
}

__device__ __forceinline__ void slot_add_h(const Lane &a, uint32_t k, uint32_t u0, long long h) {
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
      : "r"(la), "r"(ha), "r"(u0), "r"(static_cast<uint32_t>(h)),
        "r"(static_cast<uint32_t>(static_cast<unsigned long long>(h) >> 32))
      : "memory");
}

__device__ __forceinline__ void add_term(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e) {
  uint32_t k, u0;
  long long h;
  decode_fp64(lo, hi, e, k, u0, h);
  slot_add_h(a, k, u0, h);
}

// Remove exactly what add_term added for the term (lo, hi): its decode negated.
__device__ __forceinline__ void cancel_term(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e) {
  uint32_t k, u0;
  long long h;
  decode_fp64(lo, hi, e, k, u0, h);
  // -(h 2^32 + u0) = (-h - (u0 != 0)) 2^32 + (-u0 mod 2^32)
  slot_add_h(a, k, 0u - u0, -h - (u0 != 0u ? 1 : 0));
}
#else
__device__ __forceinline__ void add_term(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e) {
  uint32_t s, ep, k, la, ha, u0, u1, u2;
  decode96(lo, hi, e, s, u0, u1, u2, ep);
  asm("shr.u32 %0, %1, 5;" : "=r"(k) : "r"(ep));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(la) : "r"(k), "r"(a.c128), "r"(a.sl));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(ha) : "r"(la), "r"(a.two), "r"(a.hoff));
  asm volatile(
      "{\n\t.reg .u32 l, h0, h1, cf;\n\t"
      EXSUM_RMW_LD
      "add.cc.u32 cf, %2, %2;\n\t"
      "addc.cc.u32 l, l, %3;\n\t"
      "addc.cc.u32 h0, h0, %4;\n\t"
      "addc.u32 h1, h1, %5;\n\t"
      EXSUM_RMW_ST
      :
      : "r"(la), "r"(ha), "r"(s), "r"(u0), "r"(u1), "r"(u2)
      : "memory");
}

// Remove the blind add of an Inf/NaN term: its sign-flipped twin decodes to the
// exact negation (modular slot arithmetic).
__device__ __forceinline__ void cancel_term(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e) {
  add_term(a, lo, hi ^ 0x80000000u, e);
}
#endif

// Carry upward: L_k in [0, 2^32), H_k = 0 below the top slot, which keeps the
// rest (with 65 slots: slot 64 holds up to 2^95 units of 2^973 > any finite
// lane sum, 2^1024 x 2^31 terms).
// Safe whenever every slot has absorbed <= 2047 terms (|H_k| < 2^63 - 2^52).
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

// The warp's exact sum as 67 chunk values, straight from the (unnormalised)
// slots: slot k = L_k + 2^32 H_k feeds chunk k (L_k), chunk k+1 (low word of H_k)
// and chunk k+2 (signed high word of H_k); every addend is < 2^32 in magnitude,
// so 32-lane sums stay below 2^38.  The high word of the carry-only slot 65
// belongs to chunk 67 and is folded into chunk 66.
// Lane j sums the rows of slots j, j+32, j+64 with bank-skewed 128-bit reads
// (8 lanes per wavefront hit 8 distinct 16-byte bank groups), then the chunk
// values are assembled with shuffles: 24 LDS.128 per lane per round.

__device__ __forceinline__ void warp_chunks(unsigned char *warp_smem, int lane, long long *row) {
  __syncwarp();
  const uint32_t *Lp = reinterpret_cast<const uint32_t *>(warp_smem);
  const uint32_t *Hw = reinterpret_cast<const uint32_t *>(warp_smem + kLPlane);
  long long sl[3], shl[3], shh[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int k = 32 * r + lane;
    sl[r] = shl[r] = shh[r] = 0;
    if (k < kSlots) {
      long long a = 0, bl = 0, bh = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint4 v = *reinterpret_cast<const uint4 *>(Lp + k * 32 + 4 * ((i + lane) & 7));
        a += static_cast<long long>(v.x) + v.y + static_cast<long long>(v.z) + v.w;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint4 v = *reinterpret_cast<const uint4 *>(Hw + k * 64 + 4 * ((i + lane) & 15));
        bl += static_cast<long long>(v.x) + v.z;
        bh += static_cast<long long>(static_cast<int32_t>(v.y)) + static_cast<int32_t>(v.w);
      }
      sl[r] = a;
      shl[r] = bl;
      shh[r] = bh;
    }
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int c = 32 * r + lane;
    long long lo1 = __shfl_up_sync(0xffffffffu, shl[r], 1);   // low word sums of slot c-1
    long long hi2 = __shfl_up_sync(0xffffffffu, shh[r], 2);   // high word sums of slot c-2
    const long long wl = __shfl_sync(0xffffffffu, r ? shl[r > 0 ? r - 1 : 0] : 0ll, 31);
    const long long wh = __shfl_sync(0xffffffffu, r ? shh[r > 0 ? r - 1 : 0] : 0ll, 30 + (lane & 1));
    if (lane == 0) lo1 = wl;
    if (lane < 2) hi2 = wh;
    long long v = sl[r] + lo1 + hi2;
    if (kSlots == 66 && r == 2) {
      const long long top = __shfl_sync(0xffffffffu, shh[2], 1);  // high words of slot 65
      if (c == kChunks - 1) v += top * 4294967296ll;
    }
    if (c < kChunks) row[c] = v;
  }
}

#endif  // EXSUM_RIPPLE

// ------------------------------------------------------------- term streams

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

// ------------------------------------------------------------- term sources
//
// The stream kernels sum terms produced from their input arrays by one of:
//   kSum       x[i]                        exact_sum  (vector_ops.cpp:121-130)
//   kSqnorm    fl(x[i] * x[i])              sqnorm     (vector_ops.cpp:143-146)
//   kDot       fl(x[i] * y[i]), x, y co-aligned        dot (vector_ops.cpp:147-155)
//   kDotScalarB  the same, y read with 8-byte loads (x, y not co-aligned mod 32 B)
// Products are __dmul_rn (IEEE, round to nearest even, denormals kept: what the
// reference's SSE2 multiply computes for every non-NaN result).  A NaN product
// follows the x86 rules the reference inherits (probed on the compiled
// reference): a NaN operand propagates quieted with its payload, x first;
// 0 * Inf gives the x86 default NaN 0xFFF8000000000000.  The device product of
// those cases is a canonical NaN instead, so batches with an Inf/NaN product go
// through the fix-up, which cancels the device bits and records the x86 ones.
enum Op : int { kSum = 0, kSqnorm = 1, kDot = 2, kDotScalarB = 3 };

template <int kOp>
__device__ __forceinline__ void term_bits(uint32_t xl, uint32_t xh, uint32_t yl, uint32_t yh,
                                          uint32_t &lo, uint32_t &hi) {
  if constexpr (kOp == kSum) {
    lo = xl;
    hi = xh;
  } else {
    const double a = __hiloint2double(static_cast<int>(xh), static_cast<int>(xl));
    const double b = kOp == kSqnorm ? a : __hiloint2double(static_cast<int>(yh), static_cast<int>(yl));
    const double p = __dmul_rn(a, b);
    lo = static_cast<uint32_t>(__double2loint(p));
    hi = static_cast<uint32_t>(__double2hiint(p));
  }
}

// The bits the reference's x86 multiply produces for a*b (differs from the
// device product only when the product is a NaN).
__device__ __forceinline__ unsigned long long x86_product(unsigned long long a,
                                                          unsigned long long b) {
  const unsigned long long kAbs = 0x7FFFFFFFFFFFFFFFull, kInf = 0x7FF0000000000000ull;
  const unsigned long long kQuiet = 0x0008000000000000ull;
  if ((a & kAbs) > kInf) return a | kQuiet;
  if ((b & kAbs) > kInf) return b | kQuiet;
  const double p = __dmul_rn(__longlong_as_double(static_cast<long long>(a)),
                             __longlong_as_double(static_cast<long long>(b)));
  const unsigned long long pb = static_cast<unsigned long long>(__double_as_longlong(p));
  return (pb & kAbs) > kInf ? 0xFFF8000000000000ull : pb;  // 0 * Inf: x86 default NaN
}

// One term of a scalar head/tail (element i): Inf/NaN recorded, others added.
template <int kOp>
__device__ __forceinline__ void add_elem_checked(const Lane &a, Specials &sp, const double *x,
                                                 const double *y, unsigned long long i,
                                                 unsigned long long index) {
  const unsigned long long xb = __ldg(reinterpret_cast<const unsigned long long *>(x) + i);
  const unsigned long long yb =
      kOp >= kDot ? __ldg(reinterpret_cast<const unsigned long long *>(y) + i) : xb;
  uint32_t lo, hi;
  term_bits<kOp>(static_cast<uint32_t>(xb), static_cast<uint32_t>(xb >> 32),
                 static_cast<uint32_t>(yb), static_cast<uint32_t>(yb >> 32), lo, hi);
  const uint32_t e = exponent_field(hi);
  if (e == 0x7FFu) {
    const unsigned long long t =
        kOp == kSum ? xb : x86_product(xb, yb);
    record_special(sp, static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32), index);
  } else {
    add_term(a, lo, hi, e);
  }
}

// 256-bit streaming load (LDG.E.EF.ENL2.256): 4 terms per lane per instruction.
#if EXSUM_LDG_KIND == 1
#define EXSUM_LDG256 "ld.global.nc.v8.u32"
#elif EXSUM_LDG_KIND == 2
#define EXSUM_LDG256 "ld.global.nc.L1::evict_first.v8.u32"
#elif EXSUM_LDG_KIND == 3
#define EXSUM_LDG256 "ld.global.v8.u32"
#elif EXSUM_LDG_KIND == 4
#define EXSUM_LDG256 "ld.global.nc.L1::evict_first.L2::256B.v8.u32"
#else
#define EXSUM_LDG256 "ld.global.nc.L1::no_allocate.v8.u32"
#endif
__device__ __forceinline__ void ldg256(const double *p, uint32_t (&w)[8]) {
  asm volatile(
      EXSUM_LDG256 " {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7])
      : "l"(p));
}

// Four 8-byte loads of a 32-byte group that is only 8-byte aligned (kDotScalarB's
// y); L1-allocating so a warp's four instructions share the lines.
__device__ __forceinline__ void ldg4x64(const double *p, uint32_t (&w)[8]) {
  const unsigned long long *q = reinterpret_cast<const unsigned long long *>(p);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned long long v = __ldg(q + i);
    w[2 * i] = static_cast<uint32_t>(v);
    w[2 * i + 1] = static_cast<uint32_t>(v >> 32);
  }
}

template <int V, int kOp = kSum>
struct Batch {
  uint32_t w[V][8];                       // x
  uint32_t y[kOp >= kDot ? V : 1][8];     // y (dot only)
};

// Vector u of a batch: x (and y) of the 32-byte group `vec`.
template <int V, int kOp>
__device__ __forceinline__ void load_vec(Batch<V, kOp> &b, int u, const double *X4,
                                         const double *Y4, long long vec) {
  ldg256(X4 + 4 * vec, b.w[u]);
  if constexpr (kOp == kDot) ldg256(Y4 + 4 * vec, b.y[u]);
  if constexpr (kOp == kDotScalarB) ldg4x64(Y4 + 4 * vec, b.y[u]);
}

template <int V, int kOp>
__device__ __forceinline__ void zero_vec(Batch<V, kOp> &b, int u) {
#pragma unroll
  for (int q = 0; q < 8; ++q) b.w[u][q] = 0u;
  if constexpr (kOp >= kDot) {
#pragma unroll
    for (int q = 0; q < 8; ++q) b.y[u][q] = 0u;
  }
}

// Load vector v0 + u*32 + lane (u < V) of the 32-byte vector arrays; vectors at
// or beyond vend read as zero terms (which add nothing; 0 * 0 = +0 for products).
template <int V, int kOp>
__device__ __forceinline__ void load_batch(Batch<V, kOp> &b, const double *X4, const double *Y4,
                                           long long v0, long long vend, int lane) {
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const long long v = v0 + u * 32 + lane;
    zero_vec<V, kOp>(b, u);
    if (v < vend) load_vec<V, kOp>(b, u, X4, Y4, v);
  }
}

// Bulk L2 prefetch (cp.async.bulk.prefetch.L2) of the batch-sized stretch of
// 32-byte vectors starting at vector v0, clipped to vend.  One lane issues it a
// batch ahead of the register loads; it costs no registers and no shared memory.
// kAligned: X4 is 32-byte aligned (x always is after the head peel; kDotScalarB's
// y is only 8-byte aligned).
template <int V, bool kAligned = true>
__device__ __forceinline__ void prefetch_l2(const double *X4, long long v0, long long vend) {
  if (v0 >= vend) return;
  long long nv = vend - v0;
  if (nv > V * 32) nv = V * 32;
  const uintptr_t p0 = reinterpret_cast<uintptr_t>(X4 + 4 * v0);
  if constexpr (kAligned && EXSUM_PF_ALIGNED) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0),
                 "r"(static_cast<uint32_t>(nv) * 32u)
                 : "memory");
  } else {
    const uintptr_t p1 = p0 + static_cast<uintptr_t>(nv * 32);
    const uintptr_t a0 = p0 & ~uintptr_t{15};
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0),
                 "r"(static_cast<uint32_t>((p1 - a0 + 15) & ~uintptr_t{15}))
                 : "memory");
  }
}

template <int V, int kOp>
__device__ __forceinline__ void prefetch_batch(const double *X4, const double *Y4, long long v0,
                                               long long vend) {
  prefetch_l2<V>(X4, v0, vend);
  if constexpr (kOp >= kDot) prefetch_l2<V, kOp == kDot>(Y4, v0, vend);
}

// prefetch_l2 of the aligned x stream as straight-line code: every lane
// computes the clipped size, the one bulk prefetch is predicated on lane 0
// (no branch, so no reconvergence point in the streaming loop).
template <int V>
__device__ __forceinline__ void prefetch_l2_lane0(const double *X4, long long v0, long long vend,
                                                  int lane) {
  long long nv = vend - v0;
  if (nv > V * 32) nv = V * 32;
  const uint32_t bytes = nv > 0 ? static_cast<uint32_t>(nv) * 32u : 0u;
  const uint32_t go = (lane == 0 && bytes) ? 1u : 0u;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
      "@q cp.async.bulk.prefetch.L2.global [%0], %1;\n\t}" ::"l"(
          reinterpret_cast<uintptr_t>(X4 + 4 * v0)),
      "r"(bytes), "r"(go)
      : "memory");
}

// Inf/NaN fix-up of one batch (rare): the batch's terms were added blindly;
// re-read the lane's terms, record each Inf/NaN by index and cancel its
// (garbage) contribution with its sign-flipped twin — exact in the modular slot
// arithmetic, and always before the next renormalisation.  Kept inline (an
// out-of-line call forces the lane's Specials into local memory).
//   kScan = false: compact loop, one L2 round trip per term (cold data only).
//   kScan = true:  the batch's vectors re-read at once (L1-allocating 256-bit
//                  loads, usually L1 hits) into a bitmask of Inf/NaN terms, then
//                  only the flagged terms are re-read (data with frequent specials).
template <int V, bool kScan, int kOp>
__device__ __forceinline__ void fixup_specials(const Lane &a, Specials &sp, const double *X4,
                                               const double *Y4, long long v, long long nvec,
                                               int lane, unsigned long long ib) {
  const unsigned long long *xb = reinterpret_cast<const unsigned long long *>(X4);
  const unsigned long long *yb = reinterpret_cast<const unsigned long long *>(Y4);
  if constexpr (kScan) {
    static_assert(kOp == kSum, "scanning fix-up: plain sums only");
    static_assert(4 * V <= 32, "scan mask holds one batch");
    const uint32_t *xh = reinterpret_cast<const uint32_t *>(X4);
    uint32_t mask = 0u;
#if EXSUM_FIX_L1 == 2
    // whole 32-byte vectors, L1-allocating (8 wavefronts per LDG.256 instead of
    // 8 per 4-byte high word), four at a time
    (void)xh;
#pragma unroll
    for (int h = 0; h < V; h += 4) {
      uint32_t w[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const long long vec = v + (h + u) * 32 + lane;
        if (h + u < V && vec < nvec) {
          asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(w[u][0]), "=r"(w[u][1]), "=r"(w[u][2]), "=r"(w[u][3]),
                         "=r"(w[u][4]), "=r"(w[u][5]), "=r"(w[u][6]), "=r"(w[u][7])
                       : "l"(X4 + 4 * vec));
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) w[u][j] = 0u;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          mask |= static_cast<uint32_t>(exponent_field(w[u][2 * q + 1]) == 0x7FFu)
                  << (4 * (h + u) + q);
    }
#else
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const long long vec = v + u * 32 + lane;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t hi =
            vec < nvec ? (EXSUM_FIX_L1 ? __ldg(xh + 2 * (4 * vec + q) + 1)
                                       : __ldcg(xh + 2 * (4 * vec + q) + 1))
                       : 0u;
        mask |= static_cast<uint32_t>(exponent_field(hi) == 0x7FFu) << (4 * u + q);
      }
    }
#endif
    while (mask) {
      const int i = __ffs(mask) - 1;
      mask &= mask - 1u;
      const long long vec = v + (i >> 2) * 32 + lane;
      const int q = i & 3;
      EXSUM_DCHECK(vec >= 0 && vec < nvec);
      const unsigned long long bits =
          EXSUM_FIX_L1 ? __ldg(xb + 4 * vec + q) : __ldcg(xb + 4 * vec + q);
      const uint32_t lo = static_cast<uint32_t>(bits), hi = static_cast<uint32_t>(bits >> 32);
      record_special(sp, lo, hi, ib + 4ull * static_cast<unsigned long long>(vec) + q);
      cancel_term(a, lo, hi, 0x7FFu);  // cancel the garbage add
    }
  } else {
#pragma unroll 1
    for (int u = 0; u < V; ++u) {
      const long long vec = v + u * 32 + lane;
      if (vec >= nvec) break;
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {
        const unsigned long long xv = __ldcg(xb + 4 * vec + q);
        const unsigned long long yv = kOp >= kDot ? __ldcg(yb + 4 * vec + q) : xv;
        uint32_t lo, hi;  // the bits that were added blindly
        term_bits<kOp>(static_cast<uint32_t>(xv), static_cast<uint32_t>(xv >> 32),
                       static_cast<uint32_t>(yv), static_cast<uint32_t>(yv >> 32), lo, hi);
        if (exponent_field(hi) == 0x7FFu) {
          const unsigned long long t = kOp == kSum ? xv : x86_product(xv, yv);
          record_special(sp, static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32),
                         ib + 4ull * static_cast<unsigned long long>(vec) + q);
          cancel_term(a, lo, hi, 0x7FFu);  // cancel the garbage add
        }
      }
    }
  }
}

// Products of a freshly loaded batch, in place (x words := product words), so
// that the one-slot test, the register fast path and the rolling body see
// plain terms.  Refills still load the raw inputs (load_vec<kOp>).
template <int V, int kOp>
__device__ __forceinline__ void products_in_place(Batch<V, kOp> &b) {
  if constexpr (kOp != kSum) {
#pragma unroll
    for (int u = 0; u < V; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t lo, hi;
        term_bits<kOp>(b.w[u][2 * q], b.w[u][2 * q + 1], b.y[kOp >= kDot ? u : 0][2 * q],
                       b.y[kOp >= kDot ? u : 0][2 * q + 1], lo, hi);
        b.w[u][2 * q] = lo;
        b.w[u][2 * q + 1] = hi;
      }
  }
}

// Add one batch (registers b) with rolling refill from vector nv onward.  kGuard:
// bounds-checked refills (only the last batches need it).  Returns the batch's
// maximum exponent field (2047 iff it contained an Inf/NaN term).
// kGroup > 0 (pipelined fix-up): returns instead a bitmask of the batch's groups
// of kGroup vectors that hold an Inf/NaN term (bit g: vectors g kGroup ..).
template <int V, bool kGuard, int kOp, int kGroup = 0>
__device__ __forceinline__ uint32_t batch_rolling(const Lane &a, Batch<V, kOp> &b,
                                                  const double *X4, const double *Y4,
                                                  long long nv, long long nvec, int lane) {
  static_assert(kGroup == 0 || V % kGroup == 0, "groups tile the batch");
  constexpr int G = kGroup ? kGroup : 1;
  uint32_t emax = 0, flags = 0;
#pragma unroll
  for (int u = 0; u < V; ++u) {
    uint32_t lo[4], hi[4], e[4];
    if (kGroup && u % G == 0) emax = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // terms: products already in place (products_in_place)
      lo[q] = b.w[u][2 * q];
      hi[q] = b.w[u][2 * q + 1];
      e[q] = exponent_field(hi[q]);
      emax = max(emax, e[q]);
    }
    if (kGroup && u % G == G - 1) flags |= static_cast<uint32_t>(emax == 0x7FFu) << (u / G);
#if EXSUM_RIPPLE
    uint32_t cb = 0u;
#pragma unroll
    for (int q = 0; q < 4; ++q) add_term_cb(a, lo[q], hi[q], e[q], cb);
    if (__builtin_expect(cb != 0u, 0)) ripple_fix4(a, hi, cb);
#else
#pragma unroll
    for (int q = 0; q < 4; ++q) add_term(a, lo[q], hi[q], e[q]);
#endif
    const long long vec = nv + u * 32 + lane;
    if (!kGuard || vec < nvec) {
      EXSUM_DCHECK(vec >= 0 && vec < nvec);
      load_vec<V, kOp>(b, u, X4, Y4, vec);
    } else {
      zero_vec<V, kOp>(b, u);
    }
  }
  return kGroup ? flags : emax;
}

// Pipelined Inf/NaN fix-up (plain sums): a batch whose lane saw an Inf/NaN in
// exactly one group of kGroup vectors does not stall on a re-read.  The group's
// vectors are re-loaded into registers at the batch's end and consumed one batch
// later — record by index, cancel the blind add (modular slot arithmetic, so
// the cancel may trail a renormalisation; it counts against the carry budget
// like any add: <= 4 kGroup extra adds per window).  Two or more flagged groups
// (rare) take the synchronous scanning fix-up.
template <int kGroup>
struct PendingFix {
  uint32_t w[kGroup][8];
  long long vec;  // first vector of the group (the lane's), < 0: none
};

template <int kGroup>
__device__ __forceinline__ void pending_issue(PendingFix<kGroup> &p, const double *X4,
                                              long long vec, long long nvec) {
  p.vec = vec;
#pragma unroll
  for (int j = 0; j < kGroup; ++j) {
    const long long t = vec + 32 * j;
    if (t < nvec) {
      asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(p.w[j][0]), "=r"(p.w[j][1]), "=r"(p.w[j][2]), "=r"(p.w[j][3]),
                     "=r"(p.w[j][4]), "=r"(p.w[j][5]), "=r"(p.w[j][6]), "=r"(p.w[j][7])
                   : "l"(X4 + 4 * t));
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) p.w[j][q] = 0u;
    }
  }
}

template <int kGroup>
__device__ __forceinline__ void pending_apply(PendingFix<kGroup> &p, const Lane &a, Specials &sp,
                                              unsigned long long ib) {
#pragma unroll
  for (int j = 0; j < kGroup; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t lo = p.w[j][2 * q], hi = p.w[j][2 * q + 1];
      if (exponent_field(hi) == 0x7FFu) {
        record_special(sp, lo, hi,
                       ib + 4ull * static_cast<unsigned long long>(p.vec + 32 * j) + q);
        cancel_term(a, lo, hi, 0x7FFu);
      }
    }
  p.vec = -1;
}

// Register fast path: every lane's batch lies in slot k (|sum| < 2^89 per lane):
// sum it in registers, then one read-modify-write.  Refills are unguarded.
template <int V, int kOp>
__device__ __forceinline__ void batch_uniform(const Lane &a, Batch<V, kOp> &b, const double *X4,
                                              const double *Y4, long long nv, int lane,
                                              uint32_t k, long long nvec) {
  (void)nvec;  // EXSUM_DCHECK only
  uint32_t r0 = 0, r1 = 0, r2 = 0;
#pragma unroll
  for (int u = 0; u < V; ++u) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t sg, u0, u1, u2, ep;
      decode96(b.w[u][2 * q], b.w[u][2 * q + 1], exponent_field(b.w[u][2 * q + 1]), sg, u0, u1,
               u2, ep);
      asm("{\n\t.reg .u32 cf;\n\tadd.cc.u32 cf, %3, %3;\n\taddc.cc.u32 %0, %0, %4;\n\t"
          "addc.cc.u32 %1, %1, %5;\n\taddc.u32 %2, %2, %6;\n\t}"
          : "+r"(r0), "+r"(r1), "+r"(r2)
          : "r"(sg), "r"(u0), "r"(u1), "r"(u2));
    }
    EXSUM_DCHECK(nv + u * 32 + lane < nvec);
    load_vec<V, kOp>(b, u, X4, Y4, nv + u * 32 + lane);
  }
  slot_add96(a, k, r0, r1, r2);
}

// Magnitude fast path: every lane's batch lies in slot k >= 1 (no zeros or
// denormals: e >= 32) and holds terms of one sign (neg: 0 or ~0u per lane).
// The significands are summed unsigned in registers (|sum| < 2^89), negated
// once if the lane's terms are negative, then one read-modify-write.
template <int V, int kOp>
__device__ __forceinline__ void batch_uniform_mag(const Lane &a, Batch<V, kOp> &b,
                                                  const double *X4, const double *Y4,
                                                  long long nv, int lane, uint32_t k,
                                                  uint32_t neg, long long nvec) {
  (void)nvec;  // EXSUM_DCHECK only
  uint32_t r0 = 0, r1 = 0, r2 = 0;
#pragma unroll
  for (int u = 0; u < V; ++u) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t lo = b.w[u][2 * q], hi = b.w[u][2 * q + 1];
      uint32_t t, mh, u0, u1, u2;
      asm("shr.u32 %0, %1, 20;" : "=r"(t) : "r"(hi));  // sign | e; the funnel shifts take it mod 32
      asm("lop3.b32 %0, %1, 0xFFFFF, %2, 0xEA;" : "=r"(mh) : "r"(hi), "r"(0x100000u));
      asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u0) : "r"(0u), "r"(lo), "r"(t));
      asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u1) : "r"(lo), "r"(mh), "r"(t));
      asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u2) : "r"(mh), "r"(0u), "r"(t));
      asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
          : "+r"(r0), "+r"(r1), "+r"(r2)
          : "r"(u0), "r"(u1), "r"(u2));
    }
    EXSUM_DCHECK(nv + u * 32 + lane < nvec);
    load_vec<V, kOp>(b, u, X4, Y4, nv + u * 32 + lane);
  }
  // (r ^ neg) - neg: the two's complement for a negative lane
  asm("{\n\t.reg .u32 c;\n\tsub.u32 c, 0, %3;\n\txor.b32 %0, %0, %3;\n\txor.b32 %1, %1, %3;\n\t"
      "xor.b32 %2, %2, %3;\n\tadd.cc.u32 %0, %0, c;\n\taddc.cc.u32 %1, %1, 0;\n\taddc.u32 %2, %2, 0;\n\t}"
      : "+r"(r0), "+r"(r1), "+r"(r2)
      : "r"(neg));
  slot_add96(a, k, r0, r1, r2);
}

// One-slot test for a batch: the slot of a term is its top six exponent bits
// (hi bits 25..30; e = 0 maps to slot 0 like e' = 1).  All terms share a slot
// iff the AND and the OR of their high words agree on those bits; slot 63 may
// hold Inf/NaN and never counts as uniform.  Returns the slot bits or ~0u.
// *sign: 0 if the lane's terms are all positive, ~0u if all negative, 1 if mixed.
template <int V, int kOp>
__device__ __forceinline__ uint32_t uniform_slot(const Batch<V, kOp> &b, uint32_t *sign = nullptr) {
  uint32_t hor = 0u, hand = 0xFFFFFFFFu;
#pragma unroll
  for (int u = 0; u < V; ++u)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      hor |= b.w[u][2 * q + 1];
      hand &= b.w[u][2 * q + 1];
    }
  if (sign) *sign = ((hor ^ hand) >> 31) ? 1u : static_cast<uint32_t>(static_cast<int32_t>(hor) >> 31);
  const uint32_t kbits = hor & 0x7E000000u;
  return (kbits == (hand & 0x7E000000u) && kbits != 0x7E000000u) ? (kbits >> 25) : ~0u;
}

// Accumulate the terms of elements [begin, end) into the calling warp's lane
// accumulators.  index_base is added to positions to form special-value
// indices; norm_count counts batches since the last renormalisation
// (warp-uniform).
//   V:        vectors (4 terms) per lane per batch
//   kUniform: register fast path for one-slot batches (plain sums; larger code)
//   kSplit:   separate unguarded steady-state body (larger code, fewer instrs)
//   kScan:    scanning Inf/NaN fix-up (for data with frequent specials)
//   kOp:      term source (kSum, kSqnorm, kDot, kDotScalarB); y used by dots
//   kGroup:   > 0: pipelined Inf/NaN fix-up at this group size (PendingFix)
template <int V, bool kUniform, bool kSplit, bool kScan, int kOp = kSum, int kGroup = 0>
__device__ __forceinline__ void warp_accumulate(const double *__restrict__ x,
                                                const double *__restrict__ y,
                                                unsigned long long begin, unsigned long long end,
                                                unsigned long long index_base, const Lane &a,
                                                Specials &sp, int &norm_count, int lane,
                                                long long vfirst = 0, long long vstride = 0,
                                                bool scalar_terms = true) {
  // vfirst / vstride (in 32-byte vectors): the warp's batches start at vfirst and
  // follow every vstride vectors (0: V * 32, one contiguous range); scalar_terms:
  // this warp adds the range's unaligned head and tail terms.
  constexpr int kNormEvery = 2016 / (4 * V);  // batches between renormalisations
  static_assert(kNormEvery >= 1, "batch too large for the carry budget");
  if (begin >= end) return;
  // Scalar head up to 32-byte alignment of &x[pos], scalar tail after the
  // vectors; they are added after the first batch's loads are issued so that
  // their load latency overlaps it.
  const uintptr_t addr = reinterpret_cast<uintptr_t>(x + begin);
  unsigned long long head = ((32u - (addr & 31u)) & 31u) >> 3;
  if (head > end - begin) head = end - begin;
  const unsigned long long vbeg_t = begin + head;  // first vector's term position
  const long long nvec = static_cast<long long>((end - vbeg_t) >> 2);
  const double *X4 = x + vbeg_t;                   // 32-byte aligned
  const double *Y4 = kOp >= kDot ? y + vbeg_t : X4;
  const unsigned long long tail_t = vbeg_t + 4ull * static_cast<unsigned long long>(nvec);
  auto scalars = [&]() {
    if (!scalar_terms) return;
    if (lane < static_cast<int>(head))
      add_elem_checked<kOp>(a, sp, x, y, begin + lane, index_base + begin + lane);
    if (lane < static_cast<int>(end - tail_t))
      add_elem_checked<kOp>(a, sp, x, y, tail_t + lane, index_base + tail_t + lane);
  };
  if (nvec <= 0) {
    scalars();
    return;
  }
  constexpr long long kStep = V * 32;
  const long long vs = vstride ? vstride : kStep;  // vectors between this warp's batches
  const unsigned long long ib = index_base + vbeg_t;
  if (lane == 0) {
    for (int d = 0; d <= kPrefetchBatches; ++d)
      prefetch_batch<V, kOp>(X4, Y4, vfirst + d * vs, nvec);
  }
  Batch<V, kOp> b;
  load_batch<V, kOp>(b, X4, Y4, vfirst, nvec, lane);
  scalars();
  int backoff = 0;
  static_assert(kGroup == 0 || kOp == kSum, "pipelined fix-up: plain sums only");
  constexpr int kG1 = kGroup ? kGroup : 1;
  PendingFix<kG1> pf;
  pf.vec = -1;
  auto run = [&](auto uniform_tag) {
    constexpr bool U = decltype(uniform_tag)::value;
    for (long long v = vfirst; v < nvec; v += vs) {
      const long long nv = v + vs;
      if constexpr (EXSUM_PF_PRED && kOp == kSum) {
        prefetch_l2_lane0<V>(X4, v + (kPrefetchBatches + 1) * vs, nvec, lane);
      } else {
        if (lane == 0) prefetch_batch<V, kOp>(X4, Y4, v + (kPrefetchBatches + 1) * vs, nvec);
      }
      products_in_place<V, kOp>(b);
      uint32_t emax = 0;
      const bool steady = nv + kStep <= nvec;  // next batch complete: unguarded refills
      uint32_t k = ~0u, sgn = 1u;
      if constexpr (U) {
        if (steady) {
          if (backoff > 0) {
            --backoff;
          } else {
            k = uniform_slot<V, kOp>(b, &sgn);
            if (!__all_sync(0xffffffffu, k != ~0u)) {
              k = ~0u;
              backoff = kUniformBackoff;  // wide data rarely turns uniform
            }
          }
        }
        if (k != ~0u) {
          if (EXSUM_UNIFORM_SIGNED && __all_sync(0xffffffffu, sgn != 1u && k >= 1u)) {
            batch_uniform_mag<V, kOp>(a, b, X4, Y4, nv, lane, k, sgn, nvec);
          } else {
            batch_uniform<V, kOp>(a, b, X4, Y4, nv, lane, k, nvec);
          }
        }
      }
      if (k == ~0u) {
        if (kSplit && steady) {
          emax = batch_rolling<V, false, kOp, kGroup>(a, b, X4, Y4, nv, nvec, lane);
        } else {
          emax = batch_rolling<V, true, kOp, kGroup>(a, b, X4, Y4, nv, nvec, lane);
        }
      }
      if constexpr (kGroup > 0) {
        // emax holds the flagged groups
        if (__builtin_expect(pf.vec >= 0, 0)) pending_apply<kG1>(pf, a, sp, ib);
        if (__builtin_expect(emax != 0u, 0)) {
          if ((emax & (emax - 1u)) || nv >= nvec) {
            fixup_specials<V, kScan, kOp>(a, sp, X4, Y4, v, nvec, lane, ib);
          } else {
            pending_issue<kG1>(pf, X4, v + (__ffs(emax) - 1) * kGroup * 32 + lane, nvec);
          }
        }
      } else {
        if (__builtin_expect(emax == 0x7FFu, 0))
          fixup_specials<V, kScan, kOp>(a, sp, X4, Y4, v, nvec, lane, ib);
      }
      if (++norm_count >= kNormEvery) {
        normalize(a);
        norm_count = 0;
      }
    }
  };
  if constexpr (kUniform && EXSUM_UNIFORM_DISPATCH) {
    // the first batch decides which loop this warp runs
    uint32_t sg0;
    const uint32_t k0 = uniform_slot<V, kOp>(b, &sg0);
    if (__all_sync(0xffffffffu, k0 != ~0u)) {
      run(std::true_type{});
    } else {
      run(std::false_type{});
    }
  } else {
    run(std::integral_constant<bool, kUniform>{});
  }
  if constexpr (kGroup > 0) {
    if (pf.vec >= 0) pending_apply<kG1>(pf, a, sp, ib);
  }
}

// Segmented kernel's accumulate (round 2): full batches through the UNGUARDED
// rolling body — the single-sum kernel's steady loop, 23.9 instead of 26.7
// instructions per term (no per-vector bounds test, no register zeroing) — and
// the segment's last partial batch (< V vectors per lane) through a compact
// one-vector loop.  The last full batch's refills cannot fetch the next batch
// (it is partial), so they re-read the segment's last V*32 vectors instead: in
// range, and mostly the tail the one-vector loop reads next (so they warm
// L1/L2 for it); their register copies are never added.
template <int V>
__device__ __forceinline__ void warp_accumulate_seg(const double *__restrict__ x,
                                                    unsigned long long begin,
                                                    unsigned long long end,
                                                    unsigned long long index_base, const Lane &a,
                                                    Specials &sp, int &norm_count, int lane) {
  constexpr int kNormEvery = 2016 / (4 * V);
  if (begin >= end) return;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(x + begin);
  unsigned long long head = ((32u - (addr & 31u)) & 31u) >> 3;
  if (head > end - begin) head = end - begin;
  const unsigned long long vbeg_t = begin + head;
  const long long nvec = static_cast<long long>((end - vbeg_t) >> 2);
  const double *X4 = x + vbeg_t;
  const unsigned long long tail_t = vbeg_t + 4ull * static_cast<unsigned long long>(nvec);
  const unsigned long long ib = index_base + vbeg_t;
  constexpr long long kStep = V * 32;
  const long long nfull = nvec - nvec % kStep;  // vectors in full batches
  if (lane == 0 && nvec > 0) {
    for (int d = 0; d <= kPrefetchBatches; ++d) prefetch_batch<V, kSum>(X4, X4, d * kStep, nvec);
  }
  Batch<V, kSum> b;
  if (nfull > 0) {
#pragma unroll
    for (int u = 0; u < V; ++u) load_vec<V, kSum>(b, u, X4, X4, u * 32 + lane);
  }
  // scalar head and tail terms (alignment peel), issued under the first loads
  if (lane < static_cast<int>(head))
    add_elem_checked<kSum>(a, sp, x, x, begin + lane, index_base + begin + lane);
  if (lane < static_cast<int>(end - tail_t))
    add_elem_checked<kSum>(a, sp, x, x, tail_t + lane, index_base + tail_t + lane);
  for (long long v = 0; v < nfull; v += kStep) {
    const long long nv = v + kStep;
    prefetch_l2_lane0<V>(X4, v + (kPrefetchBatches + 1) * kStep, nvec, lane);
    const long long rb = nv + kStep <= nvec ? nv : nvec - kStep;  // refill base, in range
    const uint32_t emax = batch_rolling<V, false, kSum>(a, b, X4, X4, rb, nvec, lane);
    if (__builtin_expect(emax == 0x7FFu, 0))
      fixup_specials<V, true, kSum>(a, sp, X4, X4, v, nvec, lane, ib);
    if (++norm_count >= kNormEvery) {
      normalize(a);
      norm_count = 0;
    }
  }
  if (nfull < nvec) {
    // the partial batch: <= V vectors per lane, one at a time (counts as a batch
    // against the carry budget)
    if (norm_count + 1 >= kNormEvery) {
      normalize(a);
      norm_count = 0;
    }
    ++norm_count;
#pragma unroll 1
    for (long long t = nfull + lane; t < nvec; t += 32) {
      uint32_t w[8];
      ldg256(X4 + 4 * t, w);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t e = exponent_field(w[2 * q + 1]);
        if (e == 0x7FFu) {
          record_special(sp, w[2 * q], w[2 * q + 1], ib + 4ull * static_cast<unsigned long long>(t) + q);
        } else {
          add_term(a, w[2 * q], w[2 * q + 1], e);
        }
      }
    }
  }
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// Warp-parallel carry propagation of a 67-chunk row held as v[r] = chunk
// 32 r + lane: repeated shuffle passes until no lane holds a carry (two or three
// passes for accumulated chunk sums).  On return chunks 0..65 are in [0, 2^32)
// and chunk 66 holds the signed rest; the value is unchanged.
__device__ __forceinline__ void warp_carry(long long (&v)[3], int lane) {
  const unsigned FULL = 0xffffffffu;
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
}

// Warp-parallel finalisation (all 32 lanes of one warp): the canonical form and
// rounding of exsum_core.h (SmallAccumulator::carry_propagate + round,
// small_accumulator.cpp:244-348) without a 67-step serial chain:
//   1. carry propagation by repeated shuffle passes until no lane holds a carry
//      (two or three passes for accumulated chunk sums);
//   2. canonical top / fold of a -1 top chunk via ballots;
//   3. magnitude digits of a negative value by the two's-complement rule
//      (zero below the lowest nonzero digit z, -d_z at z, ~d_i above);
//   4. lane 0 rounds a 3-digit window at the leading digit with a sticky ballot.
// row: 67 chunk values in shared memory (any representation with |c| < 2^62).
__device__ void warp_emit_v(long long v0, long long v1, long long v2, unsigned long long P,
                            unsigned long long M, unsigned long long N,
                            unsigned long long payload, double *result, exsum_partial *partial,
                            int lane);

__device__ void warp_emit(const long long *row, unsigned long long P, unsigned long long M,
                          unsigned long long N, unsigned long long payload, double *result,
                          exsum_partial *partial, int lane) {
  warp_emit_v(row[lane], row[lane + 32], lane < 3 ? row[lane + 64] : 0, P, M, N, payload, result,
              partial, lane);
}

// The same with the row already in registers (lane holds chunks lane, lane + 32, lane + 64).
__device__ void warp_emit_v(long long v0, long long v1, long long v2, unsigned long long P,
                            unsigned long long M, unsigned long long N,
                            unsigned long long payload, double *result, exsum_partial *partial,
                            int lane) {
  const unsigned FULL = 0xffffffffu;
  long long v[3] = {v0, v1, v2};
  // 1. carries: chunk i keeps its low 32 bits, passes the rest to i + 1; chunk 66 keeps all.
  warp_carry(v, lane);
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

// ------------------------------------------------- multi-GPU exchange (P2P)
//
// exsum_p2p_sum fuses parallel_exact_sum's exchange into the sum kernel: the
// last CTA of each rank writes its canonical 592-byte record into every rank's
// mailbox over peer memory (NVLink stores), publishes it with a system-scope
// flag carrying the call's epoch, waits for every rank's flag and merges the
// records in place (merge_partials, vector_ops.cpp:64-70, with index-ordered
// specials) — one launch per rank and step, no separate collective.
// Mailbox of a rank (exsum_p2p_mailbox_bytes): two record sets and two flag
// sets selected by epoch parity, so a rank that is one step ahead never writes
// into the set its peers are still reading; then an error word.
constexpr int kMaxRanks = 8;
constexpr unsigned long long kP2PTimeoutNs = 10ull * 1000 * 1000 * 1000;  // 10 s

struct GroupArgs {  // grid split into independent sums (emulated ranks); groups = 1 otherwise
  int groups;
  unsigned long long off[kMaxRanks + 1];  // groups > 1: group g sums x[off[g], off[g+1])
};

struct P2PArgs {
  int nranks;  // 0: no exchange
  int rank;    // this process's rank; group g of an emulation is rank g
  int publish_only;  // 1: publish the record and flags, skip the wait/merge (exsum_p2p_collect
                     // finishes later) — lets tests run ranks one after another
  unsigned long long epoch;
  unsigned char *mailbox[kMaxRanks];  // rank r's mailbox, mapped into this process
};

__host__ __device__ constexpr size_t p2p_flags_offset(int nranks) {
  return (2 * static_cast<size_t>(nranks) * sizeof(exsum_partial) + 255) & ~size_t{255};
}
__host__ __device__ constexpr size_t p2p_error_offset(int nranks) {
  return p2p_flags_offset(nranks) + 2 * static_cast<size_t>(nranks) * 8;
}
__host__ __device__ constexpr size_t p2p_mailbox_bytes(int nranks) {
  return (p2p_error_offset(nranks) + 8 + 255) & ~size_t{255};
}
__device__ __forceinline__ exsum_partial *p2p_record(unsigned char *mb, int nranks, int set,
                                                     int r) {
  return reinterpret_cast<exsum_partial *>(mb) + set * nranks + r;
}
__device__ __forceinline__ unsigned long long *p2p_flag(unsigned char *mb, int nranks, int set,
                                                        int r) {
  return reinterpret_cast<unsigned long long *>(mb + p2p_flags_offset(nranks)) + set * nranks + r;
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Warp 0 of a rank's last CTA: publish this rank's record (own = its slot in
// this rank's own mailbox, already written by warp_emit) to every rank, then
// (p2p_collect) wait for all ranks and merge into row/P/M/N/payload for the
// final warp_emit.  p2p_collect returns false on a timeout (a peer never
// published), after flagging the mailbox's error word.
__device__ void p2p_publish(const P2PArgs &p2p, int me, int lane) {
  const int R = p2p.nranks;
  const int set = static_cast<int>(p2p.epoch & 1);
  const unsigned long long *own = reinterpret_cast<const unsigned long long *>(
      p2p_record(p2p.mailbox[me], R, set, me));
  constexpr int kWords = sizeof(exsum_partial) / 8;  // 74
  __syncwarp();
  // 1. the record into every other rank's slot [set][me] (peer stores)
  for (int r = 0; r < R; ++r) {
    if (r == me) continue;
    unsigned long long *dst =
        reinterpret_cast<unsigned long long *>(p2p_record(p2p.mailbox[r], R, set, me));
    for (int w = lane; w < kWords; w += 32) dst[w] = __ldcg(own + w);
  }
  __threadfence_system();  // each lane's record stores are visible everywhere ...
  __syncwarp();
  // 2. ... before this rank's flag in every mailbox
  if (lane < R) st_release_sys(p2p_flag(p2p.mailbox[lane], R, set, me), p2p.epoch);
  __syncwarp();
}

__device__ bool p2p_collect(const P2PArgs &p2p, int me, long long *row, unsigned long long &P,
                            unsigned long long &M, unsigned long long &N,
                            unsigned long long &payload, int lane) {
  const int R = p2p.nranks;
  const int set = static_cast<int>(p2p.epoch & 1);
  // 3. wait for every rank's flag in the own mailbox (bounded)
  bool ok = true;
  if (lane < R) {
    const unsigned long long *f = p2p_flag(p2p.mailbox[me], R, set, lane);
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(f) != p2p.epoch) {
      if (global_ns() - t0 > kP2PTimeoutNs) {
        ok = false;
        break;
      }
      __nanosleep(64);
    }
  }
  ok = __all_sync(0xffffffffu, ok);
  __threadfence_system();  // acquire side for every lane's record reads
  if (!ok) {
    if (lane == 0)
      *reinterpret_cast<unsigned long long *>(p2p.mailbox[me] + p2p_error_offset(R)) = p2p.epoch;
    return false;
  }
  // 4. merge: chunk sums and first indices over the ranks' records
  for (int c = lane; c < kChunks; c += 32) {
    long long sum = 0;
    for (int r = 0; r < R; ++r)
      sum += static_cast<long long>(
          __ldcv(reinterpret_cast<const unsigned long long *>(p2p_record(p2p.mailbox[me], R, set, r)) + c));
    row[c] = sum;
  }
  unsigned long long Pm = ~0ull, Mm = ~0ull, Nm = ~0ull, pay = 0;
  for (int r = 0; r < R; ++r) {
    const unsigned long long *rec = reinterpret_cast<const unsigned long long *>(
        p2p_record(p2p.mailbox[me], R, set, r));
    constexpr int kTail = sizeof(exsum_small) / 8;  // first_pos_inf, first_neg_inf, first_nan, payload
    const unsigned long long pi = __ldcv(rec + kTail), ni = __ldcv(rec + kTail + 1);
    const unsigned long long qi = __ldcv(rec + kTail + 2), py = __ldcv(rec + kTail + 3);
    Pm = min(Pm, pi);
    Mm = min(Mm, ni);
    if (qi < Nm) {
      Nm = qi;
      pay = py;
    }
  }
  P = Pm;
  M = Mm;
  N = Nm;
  payload = pay;
  __syncwarp();
  return true;
}

// --------------------------------------------------------- K1w (round 2, late)
//
// Two-phase plain sum for large arrays (EXSUM_TWO_PHASE): a windowed pass, then
// the full kernel over what it left.  Lane-private slots cost 25 KB of shared
// memory per warp, so the full kernel runs 8 warps per SM; an array whose
// terms sit in a narrow exponent range (config 4: slots 29-35) needs only a
// window of 16 slots — 6.5 KB per warp, 16 warps per SM, twice the latency
// hiding (profiles/r02_window_occupancy.log).  The windowed kernel
// (exsum_wsum_kernel) gives each warp a contiguous range of whole 512-term
// batches and a window of 16 consecutive slots chosen from its first batch
// (slot k lives at k mod 16, one non-aliased carry slot above the window).
// Each batch is added blindly; if any term of it falls outside the window —
// an exponent outside, a zero, a denormal, an Inf or a NaN — the warp removes
// the whole batch again (re-read, exact negation at the same slots) and stops:
// the rest of its range is left for the full kernel, as is every range whose
// first batch does not fit or is one-slot (the full kernel's fast path).  The
// warp's window then adds its chunk sums into the workspace, and the full
// kernel, in "jobs" mode, sums the leftover ranges (plus the unaligned head
// and tail) and finalises as usual.  Bits are independent of the split.
#ifndef EXSUM_TWO_PHASE
#define EXSUM_TWO_PHASE 1
#endif
#ifndef EXSUM_TWO_PHASE_MIN
#define EXSUM_TWO_PHASE_MIN (1ull << 28)  // terms: below, the extra launch is not amortised
#endif
constexpr int kWWarps = 16;
constexpr int kWThreads = kWWarps * 32;
constexpr int kWV = 4;                       // vectors per lane per batch
constexpr int kWSlots = 17;                  // 16 aliased window slots + 1 carry slot
constexpr int kWLPlane = kWSlots * 32 * 4;
constexpr int kWWarpSmem = kWLPlane + kWSlots * 32 * 8;  // 6528 B
// Two sign planes (EXSUM_W_PLANES = 2, default): the window holds unsigned
// magnitudes, one plane per sign, so a term needs no sign complement, no
// carry-in and no exponent extraction (see add_w2).  CTA layout, 204 KB:
//   L region [0, 64 KB): warp w's positive plane at (w >> 2) 16 KB + (w & 3) 2 KB,
//     its negative plane 8 KB above (the sign bit lands there: add_w2);
//     16 window slots x 32 lanes x 4 B each
//   H region [64 KB, 192 KB): the same with doubled offsets (64-bit high parts)
//   C region [192 KB, 204 KB): per warp and sign the carry slot, L (128 B) + H (256 B)
#ifndef EXSUM_W_PLANES
#define EXSUM_W_PLANES 2
#endif
constexpr int kW2LRegion = kWWarps * 2 * 2048;
constexpr int kW2HRegion = 2 * kW2LRegion;
constexpr int kW2CSlot = 32 * 4 + 32 * 8;
constexpr int kW2Smem = kW2LRegion + kW2HRegion + kWWarps * 2 * kW2CSlot;  // 208,896 B
constexpr int kWSmem = EXSUM_W_PLANES == 2 ? kW2Smem : kWWarps * kWWarpSmem;  // 104,448 B (one plane)
constexpr long long kWStep = kWV * 32;       // vectors per warp batch
constexpr int kWNormEvery = 2016 / (4 * kWV);
constexpr int kMaxWWarps = 4096;             // jobs capacity (256 SMs)
// jobs[2 j], jobs[2 j + 1]: the j-th leftover range (element positions), j < W + 2
// after the segment-order state (OrderState, 8448 B, zero between calls) in the
// segmented layout's scratch area, so the two kinds of call can share a workspace
constexpr size_t kJobsOffset = ((sizeof(Workspace) + 255) & ~size_t{255}) + 16384;
// + one flag after the W + 2 jobs: 1 = the windowed pass did everything and rounded
constexpr size_t kTwoPhaseWsBytes =
    kJobsOffset + (2 * (kMaxWWarps + 2) + 1) * sizeof(unsigned long long);

__device__ __forceinline__ Lane lane_view_w(unsigned char *warp_smem, int lane) {
  Lane v;
  v.L = reinterpret_cast<uint32_t *>(warp_smem) + lane;
  v.H = reinterpret_cast<unsigned long long *>(warp_smem + kWLPlane) + lane;
  v.sl = static_cast<uint32_t>(__cvta_generic_to_shared(v.L));
  v.hoff = static_cast<uint32_t>(__cvta_generic_to_shared(v.H)) - 2u * v.sl;
  v.two = (blockDim.x >> 30) + 2u;
  v.c128 = v.two * 64u;
  return v;
}

// add_term at window slot (e' >> 5) mod 16: (e' & 0x1E0) * 4 = slot * 128 bytes.
// The windowed kernel is ALU-pipe bound (ncu: math-pipe throttle 1.5 per issue,
// FMA pipe mostly idle), so EXSUM_W_XOR_IMAD moves the sign complement to the
// FMA pipe as IMADs (x (2s + 1) + s), as round 1's variant did for the full kernel.
#ifndef EXSUM_W_XOR_IMAD
#define EXSUM_W_XOR_IMAD 0
#endif
__device__ __forceinline__ void decode96_w(uint32_t lo, uint32_t hi, uint32_t e, uint32_t &s,
                                           uint32_t &u0, uint32_t &u1, uint32_t &u2,
                                           uint32_t &ep) {
#if EXSUM_W_XOR_IMAD
  uint32_t d, mhi, mh, m1, lx, mx;
  asm("shr.s32 %0, %1, 31;" : "=r"(s) : "r"(hi));
  asm("max.u32 %0, %1, 1;" : "=r"(ep) : "r"(e));
  asm("mad.lo.u32 %0, %1, -1, %2;" : "=r"(d) : "r"(e), "r"(ep));
  asm("lop3.b32 %0, %1, 0xFFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x100000u));
  asm("mad.lo.u32 %0, %1, -1048576, %2;" : "=r"(mh) : "r"(d), "r"(mhi));
  asm("mad.lo.u32 %0, %1, 2, 1;" : "=r"(m1) : "r"(s));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(lx) : "r"(lo), "r"(m1), "r"(s));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(mx) : "r"(mh), "r"(m1), "r"(s));
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u0) : "r"(s), "r"(lx), "r"(ep));
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u1) : "r"(lx), "r"(mx), "r"(ep));
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u2) : "r"(mx), "r"(s), "r"(ep));
#else
  decode96(lo, hi, e, s, u0, u1, u2, ep);
#endif
}

__device__ __forceinline__ void add_term_w(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e) {
  uint32_t s, ep, km, la, ha, u0, u1, u2;
  decode96_w(lo, hi, e, s, u0, u1, u2, ep);
  asm("and.b32 %0, %1, 480;" : "=r"(km) : "r"(ep));
  asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(la) : "r"(km), "r"(a.sl));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(ha) : "r"(la), "r"(a.two), "r"(a.hoff));
  asm volatile(
      "{\n\t.reg .u32 l, h0, h1, cf;\n\t"
      EXSUM_RMW_LD
      "add.cc.u32 cf, %2, %2;\n\t"
      "addc.cc.u32 l, l, %3;\n\t"
      "addc.cc.u32 h0, h0, %4;\n\t"
      "addc.u32 h1, h1, %5;\n\t"
      EXSUM_RMW_ST
      :
      : "r"(la), "r"(ha), "r"(s), "r"(u0), "r"(u1), "r"(u2)
      : "memory");
}

// Carry through the window in real slot order kb .. kb + 15, the last carry
// into the carry slot (same invariant as normalize()).
__device__ __forceinline__ void normalize_w(const Lane &a, int kb) {
  long long c = 0;
#pragma unroll 4
  for (int i = 0; i < 16; ++i) {
    const int j = (kb + i) & 15;
    const long long u = static_cast<long long>(a.L[32 * j]) + c;
    const long long h = static_cast<long long>(a.H[32 * j]);
    a.L[32 * j] = static_cast<uint32_t>(u);
    a.H[32 * j] = 0ull;
    c = h + (u >> 32);
  }
  const long long u = static_cast<long long>(a.L[32 * 16]) + c;
  a.L[32 * 16] = static_cast<uint32_t>(u);
  a.H[32 * 16] = static_cast<unsigned long long>(static_cast<long long>(a.H[32 * 16]) + (u >> 32));
}

// The warp's window as chunk values: lane i <= 16 sums real slot kb + i
// (window slot (kb + i) mod 16; i = 16: the carry slot) and returns chunk
// kb + i of the row; lanes 17, 18 return chunks kb + 17, kb + 18.
__device__ __forceinline__ long long warp_chunks_w(unsigned char *warp_smem, int lane, int kb) {
  __syncwarp();
  const uint32_t *Lp = reinterpret_cast<const uint32_t *>(warp_smem);
  const uint32_t *Hw = reinterpret_cast<const uint32_t *>(warp_smem + kWLPlane);
  long long sl = 0, shl = 0, shh = 0;
  if (lane <= 16) {
    const int k = lane == 16 ? 16 : (kb + lane) & 15;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = *reinterpret_cast<const uint4 *>(Lp + k * 32 + 4 * ((i + lane) & 7));
      sl += static_cast<long long>(v.x) + v.y + static_cast<long long>(v.z) + v.w;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint4 v = *reinterpret_cast<const uint4 *>(Hw + k * 64 + 4 * ((i + lane) & 15));
      shl += static_cast<long long>(v.x) + v.z;
      shh += static_cast<long long>(static_cast<int32_t>(v.y)) + static_cast<int32_t>(v.w);
    }
  }
  const long long lo1 = __shfl_up_sync(0xffffffffu, shl, 1);
  const long long hi2 = __shfl_up_sync(0xffffffffu, shh, 2);
  long long v = sl + (lane >= 1 ? lo1 : 0) + (lane >= 2 ? hi2 : 0);
  return lane <= 18 ? v : 0;
}

// ---- two sign planes (EXSUM_W_PLANES = 2) ----
// A window slot holds an unsigned 96-bit magnitude sum (L: low 32 bits, H:
// high 64).  Per term (ALU: shr, and, lop3, 3 funnel shifts, max, 3 adds;
// FMA: the fit value and the two addresses), against the one-plane decode's
// sign mask, implicit-bit and denormal handling and sign complement:
//   sh = hi >> 20 = s << 11 | e: shift amount (e mod 32, the funnel shifts
//        use sh mod 32) and, masked with 0x9E0, s << 11 | (e >> 5 mod 16) << 5:
//        times 4 the byte offset of the term's plane and window slot.
//   fit = 2 hi - (elo << 21): (e - elo) << 21 | mantissa bits for e >= elo, a
//        wrapped (huge) value below; the batch fits iff max(fit) <= lim.
// Window slots hold exponent fields e >= 32 only (kb >= 1): normal terms, so
// the implicit bit is always set.
struct WLane2 {
  uint32_t sl;    // shared address of this lane's positive-plane slot 0 (L)
  uint32_t hoff;  // H address = 2 L address + hoff
  uint32_t two;   // 2 and 4, opaque to ptxas (IMADs on the FMA pipe)
  uint32_t four;
  uint32_t *L;             // generic: positive plane slot 0, slot k at L[32 k], negative at +2048
  unsigned long long *H;   // the same for H (negative at +2048)
  uint32_t *CL;            // carry slot of the positive plane, negative at +96 words
  unsigned long long *CH;  // its H words, negative at +48
};

__device__ __forceinline__ WLane2 lane_view_w2(unsigned char *smem, int warp, int lane) {
  WLane2 v;
  const int loff = (warp >> 2) * 16384 + (warp & 3) * 2048 + lane * 4;
  v.L = reinterpret_cast<uint32_t *>(smem + loff);
  v.H = reinterpret_cast<unsigned long long *>(smem + kW2LRegion + 2 * loff);
  unsigned char *c = smem + kW2LRegion + kW2HRegion + warp * 2 * kW2CSlot;
  v.CL = reinterpret_cast<uint32_t *>(c) + lane;
  v.CH = reinterpret_cast<unsigned long long *>(c + 128) + lane;
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  v.sl = base + static_cast<uint32_t>(loff);
  v.hoff = base + static_cast<uint32_t>(kW2LRegion) - 2u * base;
  v.two = (blockDim.x >> 30) + 2u;
  v.four = v.two + v.two;
  return v;
}

// Zero the warp's planes and carry slots.
__device__ __forceinline__ void zero_w2(unsigned char *smem, int warp, int lane) {
  const int l0 = (warp >> 2) * 16384 + (warp & 3) * 2048;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    uint4 *pl = reinterpret_cast<uint4 *>(smem + l0 + s * 8192);
    uint4 *ph = reinterpret_cast<uint4 *>(smem + kW2LRegion + 2 * (l0 + s * 8192));
#pragma unroll
    for (int i = lane; i < 128; i += 32) pl[i] = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int i = lane; i < 256; i += 32) ph[i] = make_uint4(0, 0, 0, 0);
  }
  uint4 *pc = reinterpret_cast<uint4 *>(smem + kW2LRegion + kW2HRegion + warp * 2 * kW2CSlot);
  for (int i = lane; i < 2 * kW2CSlot / 16; i += 32) pc[i] = make_uint4(0, 0, 0, 0);
}

// The term (lo, hi) added to (kSub: subtracted from) its plane's window slot;
// returns the fit value.
template <bool kSub>
__device__ __forceinline__ uint32_t add_w2(const WLane2 &a, uint32_t lo, uint32_t hi,
                                           uint32_t neg_elo21) {
  uint32_t fit, sh, t, mhi, u0, u1, u2, la, ha;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(fit) : "r"(hi), "r"(a.two), "r"(neg_elo21));
  asm("shr.u32 %0, %1, 20;" : "=r"(sh) : "r"(hi));
  asm("and.b32 %0, %1, 2528;" : "=r"(t) : "r"(sh));  // 0x9E0
  asm("lop3.b32 %0, %1, 0xFFFFF, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x100000u));
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u0) : "r"(0u), "r"(lo), "r"(sh));
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u1) : "r"(lo), "r"(mhi), "r"(sh));
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(u2) : "r"(mhi), "r"(0u), "r"(sh));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(la) : "r"(t), "r"(a.four), "r"(a.sl));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(ha) : "r"(la), "r"(a.two), "r"(a.hoff));
  if constexpr (kSub) {
    asm volatile(
        "{\n\t.reg .u32 l, h0, h1;\n\t" EXSUM_RMW_LD
        "sub.cc.u32 l, l, %2;\n\t"
        "subc.cc.u32 h0, h0, %3;\n\t"
        "subc.u32 h1, h1, %4;\n\t" EXSUM_RMW_ST
        :
        : "r"(la), "r"(ha), "r"(u0), "r"(u1), "r"(u2)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .u32 l, h0, h1;\n\t" EXSUM_RMW_LD
        "add.cc.u32 l, l, %2;\n\t"
        "addc.cc.u32 h0, h0, %3;\n\t"
        "addc.u32 h1, h1, %4;\n\t" EXSUM_RMW_ST
        :
        : "r"(la), "r"(ha), "r"(u0), "r"(u1), "r"(u2)
        : "memory");
  }
  return fit;
}

// Carry each plane through real slots kb .. kb + 15 into its carry slot
// (unsigned: every slot sum stays below 2^96, normalize every kWNormEvery batches).
__device__ __forceinline__ void normalize_w2(const WLane2 &a, int kb) {
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    uint32_t *L = a.L + s * 2048;
    unsigned long long *H = a.H + s * 2048;
    unsigned long long c = 0;
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
      const int j = (kb + i) & 15;
      const unsigned long long u = static_cast<unsigned long long>(L[32 * j]) + c;
      const unsigned long long h = H[32 * j];
      L[32 * j] = static_cast<uint32_t>(u);
      H[32 * j] = 0ull;
      c = h + (u >> 32);
    }
    uint32_t *CL = a.CL + s * 96;
    unsigned long long *CH = a.CH + s * 48;
    const unsigned long long u = static_cast<unsigned long long>(*CL) + c;
    *CL = static_cast<uint32_t>(u);
    *CH += u >> 32;
  }
}

// The warp's window as chunk values (positive minus negative plane): lane
// i <= 16 sums real slot kb + i (i = 16: the carry slot) over the 32 lanes
// and returns chunk kb + i; lanes 17, 18 return chunks kb + 17, kb + 18.
__device__ __forceinline__ long long warp_chunks_w2(unsigned char *smem, int warp, int lane,
                                                    int kb) {
  __syncwarp();
  long long sl = 0, shl = 0, shh = 0;
  if (lane <= 16) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const uint32_t *Lp, *Hp;
      if (lane == 16) {
        const unsigned char *c =
            smem + kW2LRegion + kW2HRegion + (warp * 2 + s) * kW2CSlot;
        Lp = reinterpret_cast<const uint32_t *>(c);
        Hp = reinterpret_cast<const uint32_t *>(c + 128);
      } else {
        const int l0 = (warp >> 2) * 16384 + (warp & 3) * 2048 + s * 8192 + ((kb + lane) & 15) * 128;
        Lp = reinterpret_cast<const uint32_t *>(smem + l0);
        Hp = reinterpret_cast<const uint32_t *>(smem + kW2LRegion + 2 * l0);
      }
      long long ql = 0, qhl = 0, qhh = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint4 v = *reinterpret_cast<const uint4 *>(Lp + 4 * ((i + lane) & 7));
        ql += static_cast<long long>(v.x) + v.y + static_cast<long long>(v.z) + v.w;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint4 v = *reinterpret_cast<const uint4 *>(Hp + 4 * ((i + lane) & 15));
        qhl += static_cast<long long>(v.x) + v.z;
        qhh += static_cast<long long>(v.y) + v.w;
      }
      sl += s ? -ql : ql;
      shl += s ? -qhl : qhl;
      shh += s ? -qhh : qhh;
    }
  }
  const long long lo1 = __shfl_up_sync(0xffffffffu, shl, 1);
  const long long hi2 = __shfl_up_sync(0xffffffffu, shh, 2);
  long long v = sl + (lane >= 1 ? lo1 : 0) + (lane >= 2 ? hi2 : 0);
  return lane <= 18 ? v : 0;
}

__global__ void __launch_bounds__(kWThreads, 1)
exsum_wsum_kernel(const double *__restrict__ x, unsigned long long n, Workspace *__restrict__ ws,
                  unsigned long long *__restrict__ jobs, double *result, exsum_partial *partial) {
  __shared__ int s_last;
  __shared__ long long s_row[kChunks];
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
#if EXSUM_W_PLANES != 2
  unsigned char *wsm = smem + warp * kWWarpSmem;
#endif
  asm volatile("griddepcontrol.launch_dependents;");
  const int W = static_cast<int>(gridDim.x) * kWWarps;
  const int w = static_cast<int>(blockIdx.x) * kWWarps + warp;
  // geometry: 32-byte vectors from g0; whole batches only
  const uintptr_t addr = reinterpret_cast<uintptr_t>(x);
  unsigned long long head = ((32u - (addr & 31u)) & 31u) >> 3;
  if (head > n) head = n;
  const unsigned long long g0 = head;
  const long long nvec = static_cast<long long>((n - g0) >> 2);
  const long long nb = nvec / kWStep;
  const long long vb = kWStep * ((nb * w) / W), ve = kWStep * ((nb * (w + 1)) / W);
  const double *X4 = x + g0;
  unsigned long long resume = g0 + 4ull * static_cast<unsigned long long>(vb);  // nothing done
  unsigned long long head_left = 0;  // first position of the head / tail left as a job
  unsigned long long tail_left = g0 + 4ull * static_cast<unsigned long long>(nb * kWStep);
  int kb = 0;
  bool any = false;
  if (vb < ve) {
    Batch<kWV, kSum> b;
    if (lane == 0)
      for (int d = 0; d <= kPrefetchBatches; ++d)
        prefetch_batch<kWV, kSum>(X4, X4, vb + d * kWStep, ve);
    load_batch<kWV, kSum>(b, X4, X4, vb, ve, lane);
    // the window from the first batch (none if it is one-slot: the full
    // kernel's fast path is faster there)
    uint32_t emin = 0x7FFu, emax = 0;
#pragma unroll
    for (int u = 0; u < kWV; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t e = exponent_field(b.w[u][2 * q + 1]);
        emin = min(emin, e);
        emax = max(emax, e);
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, o));
      emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    }
    const int kmin = static_cast<int>(emin >> 5), kmax = static_cast<int>(emax >> 5);
#if EXSUM_W_PLANES == 2
    // two planes: window slots from 1 up (normal terms only)
    if (kmin >= 1 && emax <= 2046 && kmax - kmin <= 12 && kmax > kmin) {
      kb = kmin - (15 - (kmax - kmin)) / 2;
      kb = kb < 1 ? 1 : (kb > 48 ? 48 : kb);
#else
    if (emin >= 1 && emax <= 2046 && kmax - kmin <= 12 && kmax > kmin) {
      kb = kmin - (15 - (kmax - kmin)) / 2;
      kb = kb < 0 ? 0 : (kb > 48 ? 48 : kb);
#endif
      // exponent fields of the window's slots; 2047 (Inf/NaN) is never inside
      // (a window at the top, kb = 48, would otherwise reach it)
      const uint32_t elo = static_cast<uint32_t>(kb) * 32u, ehi = min(elo + 511u, 2046u);
      any = true;
#if EXSUM_W_PLANES == 2
      zero_w2(smem, warp, lane);
      __syncwarp();
      const WLane2 a = lane_view_w2(smem, warp, lane);
      // fit = 2 hi - (elo << 21) <= lim  <=>  elo <= e <= ehi
      const uint32_t neg_elo21 = 0u - (elo << 21), lim = ((ehi - elo + 1u) << 21) - 1u;
      int norm_count = 0;
      long long v = vb;
      for (; v < ve; v += kWStep) {
        const long long nv = v + kWStep;
        prefetch_l2_lane0<kWV>(X4, v + (kPrefetchBatches + 1) * kWStep, ve, lane);
        uint32_t fmax = 0;
#pragma unroll
        for (int u = 0; u < kWV; ++u) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            fmax = max(fmax, add_w2<false>(a, b.w[u][2 * q], b.w[u][2 * q + 1], neg_elo21));
          const long long vec = nv + u * 32 + lane;
          if (vec < ve) {
            load_vec<kWV, kSum>(b, u, X4, X4, vec);
          } else {
            zero_vec<kWV, kSum>(b, u);
          }
        }
        if (__builtin_expect(__any_sync(0xffffffffu, fmax > lim), 0)) {
          // remove this batch again (same planes and slots) and leave the rest
          // to the full kernel
#pragma unroll 1
          for (int u = 0; u < kWV; ++u) {
            uint32_t t[8];
            ldg256(X4 + 4 * (v + u * 32 + lane), t);
#pragma unroll
            for (int q = 0; q < 4; ++q) add_w2<true>(a, t[2 * q], t[2 * q + 1], neg_elo21);
          }
          break;
        }
        if (++norm_count >= kWNormEvery) {
          normalize_w2(a, kb);
          norm_count = 0;
        }
      }
      resume = g0 + 4ull * static_cast<unsigned long long>(v);
      auto scalars = [&](unsigned long long p0, unsigned long long p1) -> unsigned long long {
        for (unsigned long long p = p0; p < p1; p += 32) {
          const unsigned long long t = p + static_cast<unsigned long long>(lane);
          const unsigned long long bits =
              t < p1 ? __ldg(reinterpret_cast<const unsigned long long *>(x) + t) : 0ull;
          const uint32_t hi = static_cast<uint32_t>(bits >> 32);
          if (!__all_sync(0xffffffffu, t >= p1 || 2u * hi + neg_elo21 <= lim)) return p;
          if (++norm_count >= kWNormEvery) {
            normalize_w2(a, kb);
            norm_count = 0;
          }
          if (t < p1) add_w2<false>(a, static_cast<uint32_t>(bits), hi, neg_elo21);
        }
        return p1;
      };
#else
      {  // clear this warp's window
        uint4 *p = reinterpret_cast<uint4 *>(wsm);
#pragma unroll 4
        for (int i = lane; i < kWWarpSmem / 16; i += 32) p[i] = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
      const Lane a = lane_view_w(wsm, lane);
      int norm_count = 0;
      long long v = vb;
      for (; v < ve; v += kWStep) {
        const long long nv = v + kWStep;
        prefetch_l2_lane0<kWV>(X4, v + (kPrefetchBatches + 1) * kWStep, ve, lane);
        uint32_t bmin = 0x7FFu, bmax = 0;
#pragma unroll
        for (int u = 0; u < kWV; ++u) {
          uint32_t lo[4], hi[4], e[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            lo[q] = b.w[u][2 * q];
            hi[q] = b.w[u][2 * q + 1];
            e[q] = exponent_field(hi[q]);
            bmin = min(bmin, e[q]);
            bmax = max(bmax, e[q]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) add_term_w(a, lo[q], hi[q], e[q]);
          const long long vec = nv + u * 32 + lane;
          if (vec < ve) {
            load_vec<kWV, kSum>(b, u, X4, X4, vec);
          } else {
            zero_vec<kWV, kSum>(b, u);
          }
        }
        if (__builtin_expect(__any_sync(0xffffffffu, bmin < elo || bmax > ehi), 0)) {
          // remove this batch again and leave the rest to the full kernel
#pragma unroll 1
          for (int u = 0; u < kWV; ++u) {
            uint32_t t[8];
            ldg256(X4 + 4 * (v + u * 32 + lane), t);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              add_term_w(a, t[2 * q], t[2 * q + 1] ^ 0x80000000u, exponent_field(t[2 * q + 1]));
          }
          break;
        }
        if (++norm_count >= kWNormEvery) {
          normalize_w(a, kb);
          norm_count = 0;
        }
      }
      resume = g0 + 4ull * static_cast<unsigned long long>(v);
      // the unaligned head (warp 0) and the tail after the last whole batch
      // (last warp) through this window when every term fits; else they stay jobs
      auto scalars = [&](unsigned long long p0, unsigned long long p1) -> unsigned long long {
        for (unsigned long long p = p0; p < p1; p += 32) {
          const unsigned long long t = p + static_cast<unsigned long long>(lane);
          const unsigned long long bits =
              t < p1 ? __ldg(reinterpret_cast<const unsigned long long *>(x) + t) : 0ull;
          const uint32_t hi = static_cast<uint32_t>(bits >> 32), e = exponent_field(hi);
          if (!__all_sync(0xffffffffu, t >= p1 || (e >= elo && e <= ehi && e >= 1u && e <= 2046u)))
            return p;
          if (++norm_count >= kWNormEvery) {
            normalize_w(a, kb);
            norm_count = 0;
          }
          if (t < p1) add_term_w(a, static_cast<uint32_t>(bits), hi, e);
        }
        return p1;
      };
#endif
      if (v == ve) {
        if (w == 0) head_left = scalars(0, g0);
        if (w == W - 1)
          tail_left = scalars(g0 + 4ull * static_cast<unsigned long long>(nb * kWStep), n);
      }
    }
  }
  // the previous grid in the stream may still read the workspace and the jobs
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (any) {
#if EXSUM_W_PLANES == 2
    const long long c = warp_chunks_w2(smem, warp, lane, kb);
#else
    const long long c = warp_chunks_w(wsm, lane, kb);
#endif
    if (lane <= 18 && c) atomicAdd(&ws->chunk[kb + lane], static_cast<unsigned long long>(c));
  }
  if (lane == 0) {
    jobs[2 * w] = resume;
    jobs[2 * w + 1] = g0 + 4ull * static_cast<unsigned long long>(ve);
    if (w == 0) {  // the unaligned head
      jobs[2 * W] = head_left;
      jobs[2 * W + 1] = g0;
    }
    if (w == W - 1) {  // the tail after the last whole batch
      jobs[2 * W + 2] = tail_left;
      jobs[2 * W + 3] = n;
    }
  }
  // Last CTA: when no job is left, round here and tell the full kernel to skip
  // (jobs[2 W + 4] = 1); the windowed pass saw no Inf/NaN (it leaves them).
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&ws->wdone, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int nj = W + 2;
  int left = 0;
  for (int j = threadIdx.x; j < nj; j += blockDim.x) left |= __ldcg(&jobs[2 * j]) < __ldcg(&jobs[2 * j + 1]);
  left = __syncthreads_or(left);
  if (threadIdx.x == 0) {
    ws->wdone = 0;
    jobs[2 * nj] = left ? 0ull : 1ull;
  }
  if (left) return;
  if (threadIdx.x < kChunks) {
    s_row[threadIdx.x] = static_cast<long long>(__ldcg(&ws->chunk[threadIdx.x]));
    ws->chunk[threadIdx.x] = 0;
  }
  __syncthreads();
  if (warp == 0) warp_emit(s_row, ~0ull, ~0ull, ~0ull, 0ull, result, partial, lane);
}

template <int kOp>
__global__ void __launch_bounds__(kThreads, 1)
exsum_sum_kernel(const double *__restrict__ x, const double *__restrict__ y, unsigned long long n,
                 unsigned long long base_index, Workspace *__restrict__ ws, int finalize,
                 double *result, exsum_partial *partial, const __grid_constant__ GroupArgs grp,
                 const __grid_constant__ P2PArgs p2p,
                 const unsigned long long *__restrict__ jobs = nullptr, int njobs = 0) {
  // jobs (two-phase sums): instead of its own split of [0, n), warp gw sums the
  // ranges [jobs[2 j], jobs[2 j + 1]) for j = gw, gw + nw, ... (exsum_wsum_kernel's
  // leftovers); everything after the accumulation is unchanged.  jobs[2 njobs] = 1:
  // the windowed pass did everything and rounded, nothing to do.
  if (jobs && __ldcg(&jobs[2 * njobs]) != 0ull) return;
  // vectors per lane per batch: a dot keeps two arrays' vectors in registers
  constexpr int V = kOp >= kDot ? EXSUM_DOT_VEC : kOp == kSqnorm ? EXSUM_SQNORM_VEC : EXSUM_VEC_PER_LANE;
  // Independent sums per CTA group (groups > 1 only when emulating ranks in one
  // cooperative launch): this CTA's group, its index and the group's grid size.
  const unsigned gctas = gridDim.x / static_cast<unsigned>(grp.groups);
  const int g = static_cast<int>(blockIdx.x / gctas);
  const unsigned bid = blockIdx.x - static_cast<unsigned>(g) * gctas;
  if (grp.groups > 1) {
    x += grp.off[g];
    if (kOp >= kDot) y += grp.off[g];
    n = grp.off[g + 1] - grp.off[g];
    base_index = grp.off[g];
    ws += g;
    result = result ? result + g : nullptr;
    partial = partial ? partial + g : nullptr;
  }
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_last;
  __shared__ unsigned long long s_spec[4];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char *wsm = warp_base(smem, warp);
  long long *scratch = reinterpret_cast<long long *>(smem + kAccSmem);
  // Programmatic dependent launch: let the next sum in the stream start its CTAs
  // on SMs this grid releases (no-op unless launched with EXSUM_SUM_OVERLAP).
  asm volatile("griddepcontrol.launch_dependents;");
  EXSUM_STAMP(0);
  // K1: contiguous per-warp ranges, boundaries on 4-term multiples.
  const unsigned long long gw = static_cast<unsigned long long>(bid) * kWarps + warp;
  const unsigned long long nw = static_cast<unsigned long long>(gctas) * kWarps;
  const unsigned long long quads = (n + 3) >> 2;
  const unsigned long long qb = quads * gw / nw, qe = quads * (gw + 1) / nw;
  const unsigned long long tb = qb * 4, te = min(qe * 4, n);
  if (lane == 0 && te > tb && !jobs) {  // start the first batches' DRAM reads before zeroing smem
    const unsigned long long tp = min(te, tb + 2ull * 4 * V * 32);
#pragma unroll
    for (int arr = 0; arr < (kOp >= kDot ? 2 : 1); ++arr) {
      const double *base = arr ? y : x;
      const uintptr_t p0 = reinterpret_cast<uintptr_t>(base + tb) & ~uintptr_t{15};
      const uintptr_t p1 = reinterpret_cast<uintptr_t>(base + tp);
      const uint32_t bytes = static_cast<uint32_t>((p1 - p0 + 15) & ~uintptr_t{15});
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0), "r"(bytes) : "memory");
    }
  }
  // jobs mode: a warp whose ranges are all empty (the windowed pass did them)
  // skips its accumulator (clear, accumulate, reduce) and adds a zero row
  bool busy = true;
  if (jobs) {
    busy = false;
    for (unsigned long long j = gw; j < static_cast<unsigned long long>(njobs); j += nw)
      busy |= jobs[2 * j] < jobs[2 * j + 1];
  }
  if (busy) zero_warp(wsm, lane);
  __syncwarp();
  const Lane a = lane_view(wsm, lane);
  Specials sp{~0ull, ~0ull, ~0ull};
  int norm_count = 0;
#if EXSUM_INTERLEAVE
  // batches dealt round-robin over the grid's warps: all warps sweep one window
  (void)tb;
  (void)te;
  if (jobs) {
#pragma unroll 1
    for (unsigned long long j = gw; busy && j < static_cast<unsigned long long>(njobs); j += nw) {
      const unsigned long long jb = jobs[2 * j], je = jobs[2 * j + 1];
      if (jb < je)
        warp_accumulate<V, EXSUM_UNIFORM_FAST != 0, true, EXSUM_SUM_SCAN != 0 && kOp == kSum,
                        kOp>(x, y, jb, je, base_index, a, sp, norm_count, lane);
    }
  } else {
    warp_accumulate<V, EXSUM_UNIFORM_FAST != 0, true, EXSUM_SUM_SCAN != 0 && kOp == kSum, kOp>(
        x, y, 0, n, base_index, a, sp, norm_count, lane,
        static_cast<long long>(gw) * V * 32, static_cast<long long>(nw) * V * 32, gw == 0);
  }
#else
  warp_accumulate<V, EXSUM_UNIFORM_FAST != 0, true, EXSUM_SUM_SCAN != 0 && kOp == kSum, kOp>(
      x, y, tb, te, base_index, a, sp, norm_count, lane);
#endif

  // K2: the warp's 67 chunk sums.
  EXSUM_STAMP(1);
  if (busy) {
    warp_chunks(wsm, lane, scratch + warp * kChunks);
  } else {
    long long *r = scratch + warp * kChunks;
    r[lane] = 0;
    r[lane + 32] = 0;
    if (lane < 3) r[lane + 64] = 0;
  }
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
  EXSUM_STAMP(2);
  if (threadIdx.x == 0) s_last = atomicAdd(&ws->done, 1u) == gctas - 1;
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
    const unsigned long long i = Nf - base_index;
    payload = __ldcg(reinterpret_cast<const unsigned long long *>(x) + i);
    if constexpr (kOp == kSqnorm) payload = x86_product(payload, payload);
    if constexpr (kOp >= kDot)
      payload = x86_product(payload, __ldcg(reinterpret_cast<const unsigned long long *>(y) + i));
    if (!finalize && lane == 0) ws->nan_payload = payload;  // first NaN so far is in this launch
  }
  if (lane == 0) ws->done = 0;
  if (!finalize) {
    // Incremental sum (exsum_cuda_accumulate): store the workspace back carried,
    // so every chunk starts the next launch below 2^32 (the top one: the signed
    // rest, |c| <= |sum| / 2^1037).  One launch adds < 2^50 per chunk, so any
    // number of launches stays inside warp_emit's |c| < 2^62 — the device form
    // of the reference's carry budget (small_accumulator.cpp:174-189), which
    // lets LargeAccumulator::add(span) run for ever (large_accumulator.cpp:28-32).
    long long v[3] = {scratch[lane], scratch[lane + 32], lane < 3 ? scratch[lane + 64] : 0};
    warp_carry(v, lane);
    ws->chunk[lane] = static_cast<unsigned long long>(v[0]);
    ws->chunk[lane + 32] = static_cast<unsigned long long>(v[1]);
    if (lane < 3) ws->chunk[lane + 64] = static_cast<unsigned long long>(v[2]);
    return;
  }
  if (p2p.nranks > 0) {
    // this rank's canonical record into its own mailbox slot, then exchange
    const int me = p2p.rank + g;
    warp_emit(scratch, ~s_spec[0], ~s_spec[1], Nf, payload, nullptr,
              p2p_record(p2p.mailbox[me], p2p.nranks, static_cast<int>(p2p.epoch & 1), me), lane);
    p2p_publish(p2p, me, lane);
    if (p2p.publish_only) return;
    unsigned long long P = 0, M = 0, N = 0, pay = 0;
    if (!p2p_collect(p2p, me, scratch, P, M, N, pay, lane)) {
      if (lane == 0 && result) *result = __longlong_as_double(0x7FF80000DEAD0000ll);
      return;
    }
    warp_emit(scratch, P, M, N, pay, result, partial, lane);
    return;
  }
  warp_emit(scratch, ~s_spec[0], ~s_spec[1], Nf, payload, result, partial, lane);
  EXSUM_STAMP(3);
}

// The wait + merge half of exsum_p2p_sum for a rank whose sum kernel ran with
// publish_only: one warp, no data.
__global__ void exsum_p2p_collect_kernel(const __grid_constant__ P2PArgs p2p, double *result,
                                         exsum_partial *partial) {
  __shared__ long long row[kChunks];
  const int lane = threadIdx.x;
  unsigned long long P = 0, M = 0, N = 0, pay = 0;
  if (!p2p_collect(p2p, p2p.rank, row, P, M, N, pay, lane)) {
    if (lane == 0 && result) *result = __longlong_as_double(0x7FF80000DEAD0000ll);
    return;
  }
  __syncwarp();
  warp_emit(row, P, M, N, pay, result, partial, lane);
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

// Longest-first claim order (LPT list scheduling) for the segmented kernel.
// Warps claim segments dynamically, so the finish is set by the last segments
// claimed; with claims one segment ahead (below) a warp may also sit on a long
// unstarted segment.  Claiming the longest first bounds both by the shortest
// segments.  Two small launches bucket the lengths by octave with 8
// sub-buckets (a coarse descending sort is enough for list scheduling):
//   hist:    per-CTA shared histograms -> global counts; the last CTA turns
//            them into descending bucket bases and re-zeroes the counts;
//   scatter: per-CTA ranks within each bucket, one global atomic per bucket
//            per CTA to reserve its range, order[base + rank] = segment.
// Order within a bucket is arbitrary, which cannot change any result (each
// segment is summed by one warp either way).
// Tail-sorted order (round 2): longest-first over the WHOLE list scatters the
// warps' concurrent segments across the array; its step time varied run to run
// (2.11-2.8 ms on config 5, with rare 4.5-7.7 ms outliers at low power, i.e.
// memory-side stalls) while index order was steady (2.18 ms) but ended on a
// long tail.  So: segments before tail_start keep index order (one key, ranks
// by CTA: a sliding, contiguous working set), and only the last
// EXSUM_SEG_TAIL x (warps in the grid) segments are claimed longest first, which
// bounds the finish by short segments.  (kSegWindows = 2: head, tail.)
#ifndef EXSUM_SEG_TAIL
#define EXSUM_SEG_TAIL 4  // tail of the claim order sorted longest first, in segments per warp
#endif
constexpr int kOrderThreads = 1024;
constexpr int kOrderBuckets = 512;
constexpr int kSegWindows = 2;  // head (index order), tail (longest first)
constexpr int kOrderKeys = kOrderBuckets * kSegWindows;
static_assert(kOrderKeys % 32 == 0, "one warp scans the keys");
constexpr unsigned long long kOrderMaxSegs = 1ull << 24;  // beyond: index order
struct OrderState {                    // zeroed by exsum_cuda_workspace_init
  unsigned int hist[kOrderKeys];       // counts (zero between calls)
  unsigned int base[kOrderKeys];       // bucket cursors of the current call
  unsigned int done;                   // hist CTAs finished (zero between calls)
  unsigned int pad_[63];
};
constexpr size_t kOrderStateOffset = (sizeof(Workspace) + 255) & ~size_t{255};
constexpr size_t kOrderOffset = kOrderStateOffset + sizeof(OrderState);  // order[] in d_ws
static_assert(kJobsOffset >= kOrderOffset, "two-phase jobs clear of the order state");
// deferred-rounding records (EXSUM_SEG_DEFER) after order[], 256-byte aligned
__host__ __device__ constexpr size_t seg_records_offset(size_t nseg) {
  return (kOrderOffset + 4 * nseg + 255) & ~size_t{255};
}

__device__ __forceinline__ int length_bucket(unsigned long long len) {
  if (len < 8) return static_cast<int>(len);
  const int msb = 63 - __clzll(static_cast<long long>(len));
  return msb * 8 + static_cast<int>((len >> (msb - 3)) & 7u);
}

// key of segment s: head segments share key 0; tail segments their length bucket
__device__ __forceinline__ int order_key(const unsigned long long *offs, unsigned long long s,
                                         unsigned long long tail_start) {
  return s < tail_start ? 0 : kOrderBuckets + length_bucket(offs[s + 1] - offs[s]);
}

__global__ void __launch_bounds__(kOrderThreads)
exsum_segment_hist_kernel(const unsigned long long *__restrict__ offs, unsigned long long nseg,
                          unsigned long long tail_start, OrderState *st) {
  __shared__ unsigned int h[kOrderKeys];
  __shared__ bool last;
  const unsigned t = threadIdx.x;
  for (unsigned k = t; k < kOrderKeys; k += kOrderThreads) h[k] = 0u;
  __syncthreads();
  // the grid covers the tail only; the head (key 0, index order) is one count
  const unsigned long long s =
      tail_start + static_cast<unsigned long long>(blockIdx.x) * kOrderThreads + t;
  if (s < nseg) atomicAdd(&h[order_key(offs, s, tail_start)], 1u);
  if (blockIdx.x == 0 && t == 0) h[0] += static_cast<unsigned int>(tail_start);
  __syncthreads();
  for (unsigned k = t; k < kOrderKeys; k += kOrderThreads)
    if (h[k]) atomicAdd(&st->hist[k], h[k]);
  __threadfence();
  __syncthreads();
  if (t == 0) last = atomicAdd(&st->done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // The totals into shared memory with one load per thread (a serial loop of
  // L2 round trips here cost ~10 us), cleared for the next call.
  static_assert(kOrderKeys <= kOrderThreads, "one key per thread");
  if (t < kOrderKeys) {
    h[t] = __ldcg(&st->hist[t]);
    st->hist[t] = 0u;
  }
  __syncthreads();
  // Claim position o runs over windows ascending and, within a window, buckets
  // descending: key(o) = (o / 512) * 512 + 511 - o % 512.  base[key(o)] = the
  // number of segments at positions before o.  One warp: lane t owns positions
  // [P t, P t + P).
  if (t < 32) {
    constexpr int P = kOrderKeys / 32;
    auto key_of = [](int o) { return (o / kOrderBuckets) * kOrderBuckets + kOrderBuckets - 1 - o % kOrderBuckets; };
    unsigned sum = 0;
    for (int i = 0; i < P; ++i) sum += h[key_of(P * t + i)];
    unsigned before = sum;  // inclusive prefix over lanes <= t
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned w = __shfl_up_sync(0xffffffffu, before, o);
      if (t >= o) before += w;
    }
    before -= sum;
    for (int i = 0; i < P; ++i) {
      const int k = key_of(P * t + i);
      st->base[k] = before;
      before += h[k];
    }
    if (t == 0) st->done = 0u;
  }
}

__global__ void __launch_bounds__(kOrderThreads)
exsum_segment_scatter_kernel(const unsigned long long *__restrict__ offs, unsigned long long nseg,
                             unsigned long long tail_start, OrderState *st,
                             unsigned int *__restrict__ order) {
  __shared__ unsigned int cnt[kOrderKeys];
  const unsigned t = threadIdx.x;
  for (unsigned k = t; k < kOrderKeys; k += kOrderThreads) cnt[k] = 0u;
  __syncthreads();
  const unsigned long long s = static_cast<unsigned long long>(blockIdx.x) * kOrderThreads + t;
  const bool head = s < tail_start;  // the head keeps index order: claim position s
  if (head) order[s] = static_cast<unsigned>(s);
  int key = 0;
  unsigned r = 0;
  if (!head && s < nseg) {
    key = order_key(offs, s, tail_start);
    r = atomicAdd(&cnt[key], 1u);
  }
  __syncthreads();
  for (unsigned k = t; k < kOrderKeys; k += kOrderThreads)
    if (cnt[k]) cnt[k] = atomicAdd(&st->base[k], cnt[k]);  // this CTA's range in bucket k
  __syncthreads();
  if (!head && s < nseg) order[cnt[key] + r] = static_cast<unsigned>(s);
}

// Lane 0's claim of the next segment: the claim atomic, the segment's entry in
// the claim order, then its offsets (three dependent round trips, straight-line).
struct SegmentClaim {
  unsigned int s;
  unsigned long long b, e;

  __device__ __forceinline__ void claim(unsigned int *counter, const unsigned int *order,
                                        const unsigned long long *offs, unsigned long long nseg) {
    unsigned int c;
    // inline PTX: a plain atomicAdd in a lane-0 branch becomes a warp-aggregated
    // atomic whose result is shuffled back at once
    asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(c) : "l"(counter) : "memory");
    s = c < nseg ? (order ? __ldcg(order + c) : c) : static_cast<unsigned int>(nseg);
    if (s < nseg) {
      b = __ldg(offs + s);
      e = __ldg(offs + s + 1);
      if (e < b) e = b;  // decreasing offsets (a caller error): an empty segment, +0.0
    }
  }
};

__global__ void __launch_bounds__(kThreads, 1)
exsum_segmented_kernel(const double *__restrict__ x, const unsigned long long *__restrict__ offs,
                       unsigned long long nseg, Workspace *__restrict__ ws, double *out,
                       exsum_partial *partials, const unsigned int *__restrict__ order,
                       exsum_partial *raw) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  long long *rows = reinterpret_cast<long long *>(smem + kAccSmem);
  long long *row = rows + warp * kChunks;
  unsigned char *wsm = warp_base(smem, warp);
  const Lane a = lane_view(wsm, lane);
  SegmentClaim ca{0u, 0ull, 0ull};
  if (lane == 0)
    ca.claim(&ws->seg_next, order, offs, nseg);  // the first claim
#if EXSUM_TIMELINE
  unsigned long long ph[7] = {0, 0, 0, 0, 0, 0, 0}, tq = gtimer(), tn;
#define EXSUM_SEG_PHASE(i) (tn = gtimer(), ph[i] += tn - tq, tq = tn)
#else
#define EXSUM_SEG_PHASE(i) ((void)0)
#endif
  EXSUM_SEG_PHASE(0);
  while (true) {
    const unsigned int s = __shfl_sync(0xffffffffu, ca.s, 0);
    if (s >= nseg) break;
    const unsigned long long b = __shfl_sync(0xffffffffu, ca.b, 0),
                             e = __shfl_sync(0xffffffffu, ca.e, 0);
#if EXSUM_SEG_AHEAD
    // claim the next segment now: its result is ready when this one ends, so
    // its head can be pulled into L2 while this segment's epilogue runs
    SegmentClaim cn{0u, 0ull, 0ull};
    if (lane == 0) cn.claim(&ws->seg_next, order, offs, nseg);
#endif
    zero_warp(wsm, lane);
    __syncwarp();
    int norm_count = 0;
    EXSUM_SEG_PHASE(1);
#if EXSUM_TIMELINE
    ph[5] += 1;
    ph[6] += e - b;
#endif
    Specials sp{~0ull, ~0ull, ~0ull};
    // indices local to the segment: position - b
#if EXSUM_SEG_SPLIT
    warp_accumulate_seg<EXSUM_SEG_VEC>(x, b, e, 0ull - b, a, sp, norm_count, lane);
#else
    warp_accumulate<EXSUM_SEG_VEC, false, false, true, kSum, EXSUM_SEG_FIX_GROUP>(
        x, x, b, e, 0ull - b, a, sp, norm_count, lane);
#endif
    EXSUM_SEG_PHASE(2);
#if EXSUM_SEG_AHEAD
    if (lane == 0) {
      ca = cn;
      if (ca.s < nseg && ca.e > ca.b) {  // the next head (<= 2 batches) into L2
        const unsigned long long hb = ca.b;
        const unsigned long long he = ca.e - hb > 2ull * 4 * 32 * EXSUM_SEG_VEC
                                          ? hb + 2ull * 4 * 32 * EXSUM_SEG_VEC
                                          : ca.e;
        const uintptr_t p0 = reinterpret_cast<uintptr_t>(x + hb) & ~uintptr_t{15};
        const uintptr_t p1 = reinterpret_cast<uintptr_t>(x + he);
        const uint32_t bytes = static_cast<uint32_t>((p1 - p0) & ~uintptr_t{15});
        if (bytes)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0), "r"(bytes)
                       : "memory");
      }
    }
#else
    if (lane == 0)
      ca.claim(&ws->seg_next, order, offs, nseg);
#endif
    EXSUM_SEG_PHASE(0);
    warp_chunks(wsm, lane, row);
#if EXSUM_SEG_PF_NEXT && !EXSUM_SEG_AHEAD
    // the claim has returned by now: start the next segment's first batches
    // towards L2 while this segment's record is written and the planes cleared
    if (lane == 0 && ca.s < nseg && ca.e > ca.b) {
      const unsigned long long hb = ca.b;
      const unsigned long long he = ca.e - hb > 2ull * 4 * 32 * EXSUM_SEG_VEC
                                        ? hb + 2ull * 4 * 32 * EXSUM_SEG_VEC
                                        : ca.e;
      const uintptr_t p0 = (reinterpret_cast<uintptr_t>(x + hb) + 15) & ~uintptr_t{15};
      const uintptr_t p1 = reinterpret_cast<uintptr_t>(x + he) & ~uintptr_t{15};
      if (p1 > p0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0),
                     "r"(static_cast<uint32_t>(p1 - p0))
                     : "memory");
    }
#endif
    const unsigned long long P = warp_min_u64(sp.P), M = warp_min_u64(sp.M),
                             N = warp_min_u64(sp.N);
    __syncwarp();
    EXSUM_SEG_PHASE(3);
    if (raw) {
      // deferred: the raw chunk sums and first indices; exsum_segment_emit_kernel
      // canonicalises and rounds every segment after this launch
      long long *dst = reinterpret_cast<long long *>(raw[s].acc.chunk);
      dst[lane] = row[lane];
      dst[lane + 32] = row[lane + 32];
      if (lane < 3) {
        dst[lane + 64] = row[lane + 64];
        reinterpret_cast<unsigned long long *>(&raw[s].first_pos_inf)[lane] =
            lane == 0 ? P : lane == 1 ? M : N;
      }
    } else {
      const unsigned long long payload =
          N != ~0ull ? __ldg(reinterpret_cast<const unsigned long long *>(x) + b + N) : 0ull;
      warp_emit(row, P, M, N, payload, out + s, partials ? partials + s : nullptr, lane);
    }
    __syncwarp();
    EXSUM_SEG_PHASE(4);
  }
#if EXSUM_TIMELINE
  if (lane == 0 && blockIdx.x < 148)
    for (int i = 0; i < 7; ++i) g_seg_timeline[(blockIdx.x * kWarps + warp) * 8 + i] = ph[i];
#endif
#undef EXSUM_SEG_PHASE
  // Last warp out resets the claim counters for the next launch.
  if (lane == 0) {
    const unsigned int total = gridDim.x * kWarps;
    __threadfence();
    if (atomicAdd(&ws->seg_done, 1u) == total - 1) {
      ws->seg_next = 0;
      ws->seg_done = 0;
    }
  }
}

// Second half of a deferred segmented sum: one warp per segment canonicalises
// its raw record (chunk sums |c| < 2^44, local first indices) and rounds it —
// the per-segment warp_emit taken off the streaming warps.  raw may alias
// partials (in place: every lane's loads precede the warp's stores).
constexpr int kEmitWarps = 8;
__global__ void __launch_bounds__(32 * kEmitWarps)
exsum_segment_emit_kernel(const exsum_partial *raw, const unsigned long long *__restrict__ offs,
                          const double *__restrict__ x, unsigned long long nseg, double *out,
                          exsum_partial *partials) {
  const int lane = threadIdx.x & 31;
  const unsigned long long s =
      static_cast<unsigned long long>(blockIdx.x) * kEmitWarps + (threadIdx.x >> 5);
  if (s >= nseg) return;
  const long long *c = reinterpret_cast<const long long *>(raw[s].acc.chunk);
  const long long v0 = __ldcg(c + lane), v1 = __ldcg(c + lane + 32),
                  v2 = lane < 3 ? __ldcg(c + lane + 64) : 0;
  const unsigned long long *f = reinterpret_cast<const unsigned long long *>(&raw[s].first_pos_inf);
  const unsigned long long P = __ldcg(f), M = __ldcg(f + 1), N = __ldcg(f + 2);
  const unsigned long long payload =
      N != ~0ull ? __ldg(reinterpret_cast<const unsigned long long *>(x) + offs[s] + N) : 0ull;
  __syncwarp();
  warp_emit_v(v0, v1, v2, P, M, N, payload, out + s, partials ? partials + s : nullptr, lane);
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
std::atomic<int> g_num_sms[kMaxDevices] = {};  // 0 = not configured yet
std::mutex g_configure_mutex;

// Per-device one-time setup: SM count and the >48 KB dynamic smem opt-in.
// Thread-safe: the fast path is one atomic load; first use takes a mutex.
int prepare_device(int *sms) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return EXSUM_ECUDA;
  int ready = g_num_sms[dev].load(std::memory_order_acquire);
  if (ready > 0) {
    *sms = ready;
    return EXSUM_OK;
  }
  std::lock_guard<std::mutex> lock(g_configure_mutex);
  if (g_num_sms[dev].load(std::memory_order_relaxed) == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      return EXSUM_ECUDA;
    if (cudaFuncSetAttribute(exsum_sum_kernel<kSum>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmem) != cudaSuccess ||
        cudaFuncSetAttribute(exsum_sum_kernel<kSqnorm>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) != cudaSuccess ||
        cudaFuncSetAttribute(exsum_sum_kernel<kDot>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmem) != cudaSuccess ||
        cudaFuncSetAttribute(exsum_sum_kernel<kDotScalarB>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) != cudaSuccess ||
        cudaFuncSetAttribute(exsum_segmented_kernel,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) != cudaSuccess ||
        cudaFuncSetAttribute(exsum_wsum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kWSmem) != cudaSuccess ||
        // the same (maximal) shared-memory carveout as the full kernel: no L1/smem
        // reconfiguration between the two phases
        cudaFuncSetAttribute(exsum_wsum_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             100) != cudaSuccess)
      return EXSUM_ECUDA;
    g_num_sms[dev].store(n, std::memory_order_release);
  }
  *sms = g_num_sms[dev].load(std::memory_order_relaxed);
  return EXSUM_OK;
}

int launch_status() { return cudaGetLastError() == cudaSuccess ? EXSUM_OK : EXSUM_ECUDA; }

// Grid for a sum of n terms: one CTA per SM, fewer for small inputs (keep at
// least ~4 K terms per warp so the per-CTA fixed cost stays amortised).
#ifndef EXSUM_MAX_CTAS
#define EXSUM_MAX_CTAS 0  // experiment: cap the sum grid below the SM count (0 = no cap)
#endif
#ifndef EXSUM_OVERLAP_SHORT
#define EXSUM_OVERLAP_SHORT 150000000ull  // overlapped sums up to this many terms leave SMs free
#endif
// Overlapped (programmatic dependent launch) sums of up to EXSUM_OVERLAP_SHORT
// terms run on 8/9 of the SMs: the free SMs let the next sum in the stream start
// streaming while this one drains, which outweighs their share of a short sum
// (config 2 sustained +4%, 30 M terms +20%); longer or non-overlapped sums use
// every SM (profiles/r01_grid_sweep.log).
unsigned grid_for(unsigned long long n, int sms, bool overlap = false) {
  if (EXSUM_MAX_CTAS > 0 && sms > EXSUM_MAX_CTAS) sms = EXSUM_MAX_CTAS;
  if (overlap && n <= EXSUM_OVERLAP_SHORT) sms -= sms / 9;
  const unsigned long long per_cta = 4096ull * kWarps;
  unsigned long long g = (n + per_cta - 1) / per_cta;
  if (g < 1) g = 1;
  if (g > static_cast<unsigned long long>(sms)) g = sms;
  return static_cast<unsigned>(g);
}

int sum_launch(const double *d_x, size_t n, uint64_t base_index, void *d_ws, size_t ws_bytes,
               void *stream, int finalize, double *d_result, exsum_partial *d_partial,
               unsigned flags = 0, int op = kSum, const double *d_y = nullptr,
               const P2PArgs *p2p = nullptr, const GroupArgs *grp = nullptr,
               bool cooperative = false, unsigned max_ctas = 0) {
  if (!d_ws || ws_bytes < sizeof(Workspace) || (n && !d_x) || (op >= kDot && n && !d_y))
    return EXSUM_EINVAL;
  int sms = 0;
  const int st = prepare_device(&sms);
  if (st) return st;
  GroupArgs g1 = {};
  g1.groups = 1;
  const GroupArgs G = grp ? *grp : g1;
  const P2PArgs X = p2p ? *p2p : P2PArgs{};
  cudaLaunchConfig_t cfg = {};
  // emulated ranks: the whole SM set split into equal co-resident groups
  if (max_ctas && static_cast<unsigned>(sms) > max_ctas) sms = static_cast<int>(max_ctas);
  cfg.gridDim = dim3(G.groups > 1 ? (sms / G.groups) * G.groups
                                   : grid_for(n, sms, (flags & EXSUM_SUM_OVERLAP) != 0));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (flags & EXSUM_SUM_OVERLAP) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cooperative) {  // CTAs wait on one another: all must be resident
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = na ? attr : nullptr;
  cfg.numAttrs = na;
  const unsigned long long nn = n, bi = base_index;
  Workspace *ws = static_cast<Workspace *>(d_ws);
  cudaError_t e;
  if (EXSUM_TWO_PHASE && op == kSum && finalize && X.nranks == 0 && G.groups == 1 &&
      !cooperative && !max_ctas && n >= EXSUM_TWO_PHASE_MIN && ws_bytes >= kTwoPhaseWsBytes &&
      sms * kWWarps <= kMaxWWarps) {
    // two-phase: the windowed pass (PDL like a plain sum), then the full kernel
    // over its leftovers in stream order
    auto *jobs = reinterpret_cast<unsigned long long *>(static_cast<unsigned char *>(d_ws) +
                                                        kJobsOffset);
    cudaLaunchConfig_t wc = cfg;
    wc.gridDim = dim3(static_cast<unsigned>(sms));
    wc.blockDim = dim3(kWThreads);
    wc.dynamicSmemBytes = kWSmem;
    e = cudaLaunchKernelEx(&wc, exsum_wsum_kernel, d_x, nn, ws, jobs, d_result, d_partial);
    if (e != cudaSuccess) return EXSUM_ECUDA;
    cudaLaunchConfig_t rc = cfg;
    rc.gridDim = dim3(static_cast<unsigned>(sms));
    rc.attrs = nullptr;
    rc.numAttrs = 0;
    const unsigned long long *cj = jobs;
    const int nj = sms * kWWarps + 2;
    e = cudaLaunchKernelEx(&rc, exsum_sum_kernel<kSum>, d_x, d_x, nn, bi, ws, finalize, d_result,
                           d_partial, G, X, cj, nj);
    if (e != cudaSuccess) return EXSUM_ECUDA;
    return launch_status();
  }
  const unsigned long long *no_jobs = nullptr;
  switch (op) {
    case kSqnorm:
      e = cudaLaunchKernelEx(&cfg, exsum_sum_kernel<kSqnorm>, d_x, d_x, nn, bi, ws, finalize,
                             d_result, d_partial, G, X, no_jobs, 0);
      break;
    case kDot:
      e = cudaLaunchKernelEx(&cfg, exsum_sum_kernel<kDot>, d_x, d_y, nn, bi, ws, finalize,
                             d_result, d_partial, G, X, no_jobs, 0);
      break;
    case kDotScalarB:
      e = cudaLaunchKernelEx(&cfg, exsum_sum_kernel<kDotScalarB>, d_x, d_y, nn, bi, ws, finalize,
                             d_result, d_partial, G, X, no_jobs, 0);
      break;
    default:
      e = cudaLaunchKernelEx(&cfg, exsum_sum_kernel<kSum>, d_x, d_x, nn, bi, ws, finalize,
                             d_result, d_partial, G, X, no_jobs, 0);
  }
  if (e != cudaSuccess) return EXSUM_ECUDA;
  return launch_status();
}

int dot_op(const double *d_a, const double *d_b) {
  return ((reinterpret_cast<uintptr_t>(d_a) ^ reinterpret_cast<uintptr_t>(d_b)) & 31u) == 0
             ? kDot
             : kDotScalarB;
}

}  // namespace

extern "C" {

uint64_t exsum_cuda_two_phase_min(void) { return EXSUM_TWO_PHASE ? EXSUM_TWO_PHASE_MIN : 0; }

size_t exsum_cuda_workspace_bytes(void) {
  // room for the two-phase sum's job list (large plain sums); sizeof(Workspace)
  // is the minimum every entry point accepts
  return EXSUM_TWO_PHASE ? kTwoPhaseWsBytes : sizeof(Workspace);
}

int exsum_cuda_workspace_init(void *d_ws, size_t ws_bytes, void *stream) {
  if (!d_ws || ws_bytes < sizeof(Workspace)) return EXSUM_EINVAL;
  // the segment-order state too when the workspace has room for it
  const size_t z = ws_bytes >= kOrderOffset ? kOrderOffset : sizeof(Workspace);
  return cudaMemsetAsync(d_ws, 0, z, static_cast<cudaStream_t>(stream)) ==
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
  EXSUM_NVTX("exsum_cuda_sum");
  return sum_launch(d_x, n, base_index, d_ws, ws_bytes, stream, 1, d_result, d_partial, flags);
}

int exsum_cuda_sum_cfg(const double *d_x, size_t n, uint64_t base_index, double *d_result,
                       exsum_partial *d_partial, void *d_ws, size_t ws_bytes, void *stream,
                       const exsum_launch_config *cfg) {
  EXSUM_NVTX("exsum_cuda_sum");
  if (cfg && (cfg->flags & ~EXSUM_SUM_OVERLAP)) return EXSUM_EINVAL;
  return sum_launch(d_x, n, base_index, d_ws, ws_bytes, stream, 1, d_result, d_partial,
                    cfg ? cfg->flags : 0u, kSum, nullptr, nullptr, nullptr, false,
                    cfg ? cfg->max_ctas : 0u);
}

int exsum_cuda_sqnorm(const double *d_x, size_t n, uint64_t base_index, double *d_result,
                      exsum_partial *d_partial, void *d_ws, size_t ws_bytes, void *stream) {
  EXSUM_NVTX("exsum_cuda_sqnorm");
  return sum_launch(d_x, n, base_index, d_ws, ws_bytes, stream, 1, d_result, d_partial, 0,
                    kSqnorm);
}

int exsum_cuda_dot(const double *d_a, size_t na, const double *d_b, size_t nb,
                   uint64_t base_index, double *d_result, exsum_partial *d_partial, void *d_ws,
                   size_t ws_bytes, void *stream) {
  EXSUM_NVTX("exsum_cuda_dot");
  if (na != nb) return EXSUM_EINVAL;  // dot: length mismatch (vector_ops.cpp:150-152)
  return sum_launch(d_a, na, base_index, d_ws, ws_bytes, stream, 1, d_result, d_partial, 0,
                    dot_op(d_a, d_b), d_b);
}

size_t exsum_p2p_mailbox_bytes(int nranks) {
  return nranks < 1 || nranks > kMaxRanks ? 0 : p2p_mailbox_bytes(nranks);
}

int exsum_p2p_mailbox_alloc(int nranks, void **d_mailbox) {
  if (!d_mailbox || nranks < 1 || nranks > kMaxRanks) return EXSUM_EINVAL;
  *d_mailbox = nullptr;
  const size_t bytes = p2p_mailbox_bytes(nranks);
  if (cudaMalloc(d_mailbox, bytes) != cudaSuccess) return EXSUM_ENOMEM;
  if (cudaMemset(*d_mailbox, 0, bytes) != cudaSuccess) {
    cudaFree(*d_mailbox);
    *d_mailbox = nullptr;
    return EXSUM_ECUDA;
  }
  return EXSUM_OK;
}

int exsum_p2p_mailbox_free(void *d_mailbox) {
  if (!d_mailbox) return EXSUM_EINVAL;
  return cudaFree(d_mailbox) == cudaSuccess ? EXSUM_OK : EXSUM_ECUDA;
}

int exsum_p2p_sum(const double *d_shard, size_t n, uint64_t base_index, int rank, int nranks,
                  void *const *mailboxes, uint64_t epoch, double *d_result,
                  exsum_partial *d_partial, void *d_ws, size_t ws_bytes, void *stream,
                  unsigned flags) {
  EXSUM_NVTX("exsum_p2p_sum");
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || !mailboxes || epoch == 0)
    return EXSUM_EINVAL;
  P2PArgs X = {};
  X.nranks = nranks;
  X.rank = rank;
  X.epoch = epoch;
  X.publish_only = (flags & EXSUM_P2P_PUBLISH_ONLY) ? 1 : 0;
  for (int r = 0; r < nranks; ++r) {
    if (!mailboxes[r]) return EXSUM_EINVAL;
    X.mailbox[r] = static_cast<unsigned char *>(mailboxes[r]);
  }
  return sum_launch(d_shard, n, base_index, d_ws, ws_bytes, stream, 1, d_result, d_partial,
                    flags & ~EXSUM_P2P_PUBLISH_ONLY, kSum, nullptr, &X);
}

int exsum_p2p_collect(int rank, int nranks, void *const *mailboxes, uint64_t epoch,
                      double *d_result, exsum_partial *d_partial, void *stream) {
  EXSUM_NVTX("exsum_p2p_collect");
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || !mailboxes || epoch == 0)
    return EXSUM_EINVAL;
  P2PArgs X = {};
  X.nranks = nranks;
  X.rank = rank;
  X.epoch = epoch;
  for (int r = 0; r < nranks; ++r) {
    if (!mailboxes[r]) return EXSUM_EINVAL;
    X.mailbox[r] = static_cast<unsigned char *>(mailboxes[r]);
  }
  exsum_p2p_collect_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(X, d_result,
                                                                          d_partial);
  return cudaGetLastError() == cudaSuccess ? EXSUM_OK : EXSUM_ECUDA;
}

int exsum_p2p_emulate_sum(const double *d_x, const uint64_t *bounds, int nranks, uint64_t epoch,
                          double *d_results, exsum_partial *d_partials, void *d_mailboxes,
                          void *d_ws, size_t ws_bytes, void *stream) {
  if (nranks < 1 || nranks > kMaxRanks || !bounds || !d_mailboxes || !d_ws || epoch == 0 ||
      ws_bytes < nranks * sizeof(Workspace))
    return EXSUM_EINVAL;
  GroupArgs G = {};
  G.groups = nranks;
  P2PArgs X = {};
  X.nranks = nranks;
  X.rank = 0;
  X.epoch = epoch;
  for (int r = 0; r <= nranks; ++r) {
    if (r && bounds[r] < bounds[r - 1]) return EXSUM_EINVAL;
    G.off[r] = bounds[r];
  }
  for (int r = 0; r < nranks; ++r)
    X.mailbox[r] = static_cast<unsigned char *>(d_mailboxes) + r * p2p_mailbox_bytes(nranks);
  return sum_launch(d_x, bounds[nranks] - bounds[0], bounds[0], d_ws, sizeof(Workspace), stream,
                    1, d_results, d_partials, 0, kSum, nullptr, &X, &G, true);
}

int exsum_p2p_error(const void *d_mailbox, int nranks, uint64_t *epoch_out, void *stream) {
  if (!d_mailbox || !epoch_out || nranks < 1 || nranks > kMaxRanks) return EXSUM_EINVAL;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(epoch_out, static_cast<const unsigned char *>(d_mailbox) +
                                     p2p_error_offset(nranks),
                      8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return EXSUM_ECUDA;
  return EXSUM_OK;
}

int exsum_ipc_get_handle(const void *d_ptr, void *handle) {
  if (!d_ptr || !handle) return EXSUM_EINVAL;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void *>(d_ptr)) != cudaSuccess) return EXSUM_ECUDA;
  memcpy(handle, &h, sizeof h);
  return EXSUM_OK;
}

int exsum_ipc_open(const void *handle, void **d_ptr) {
  if (!handle || !d_ptr) return EXSUM_EINVAL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  return cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess
             ? EXSUM_OK
             : EXSUM_ECUDA;
}

int exsum_ipc_close(void *d_ptr) {
  if (!d_ptr) return EXSUM_EINVAL;
  return cudaIpcCloseMemHandle(d_ptr) == cudaSuccess ? EXSUM_OK : EXSUM_ECUDA;
}

int exsum_cuda_accumulate(const double *d_x, size_t n, uint64_t base_index, void *d_ws,
                          size_t ws_bytes, void *stream) {
  EXSUM_NVTX("exsum_cuda_accumulate");
  if (n == 0) return (d_ws && ws_bytes >= sizeof(Workspace)) ? EXSUM_OK : EXSUM_EINVAL;
  return sum_launch(d_x, n, base_index, d_ws, ws_bytes, stream, 0, nullptr, nullptr);
}

int exsum_cuda_finalize(double *d_result, exsum_partial *d_partial, void *d_ws, size_t ws_bytes,
                        void *stream) {
  EXSUM_NVTX("exsum_cuda_finalize");
  if (!d_ws || ws_bytes < sizeof(Workspace)) return EXSUM_EINVAL;
  exsum_finalize_kernel<<<1, 96, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<Workspace *>(d_ws), d_result, d_partial);
  return launch_status();
}

int exsum_cuda_sum_segmented(const double *d_x, const uint64_t *d_offsets, size_t nseg,
                             double *d_out, exsum_partial *d_partials, void *d_ws,
                             size_t ws_bytes, void *stream) {
  EXSUM_NVTX("exsum_cuda_sum_segmented");
  if (!d_ws || ws_bytes < sizeof(Workspace) || (nseg && (!d_offsets || !d_out)))
    return EXSUM_EINVAL;
  if (nseg == 0) return EXSUM_OK;
  if (nseg >= 0xFFFFFFFFull) return EXSUM_EINVAL;
  int sms = 0;
  const int st = prepare_device(&sms);
  if (st) return st;
  unsigned long long g = (nseg + kWarps - 1) / kWarps;
  if (g > static_cast<unsigned long long>(sms)) g = sms;
  const auto *offs = reinterpret_cast<const unsigned long long *>(d_offsets);
  // Longest-first claim order when the caller's workspace has room for it and
  // there are more segments than warps (otherwise every warp gets at most one).
  unsigned int *order = nullptr;
  if (ws_bytes >= exsum_cuda_segmented_workspace_bytes(nseg) && nseg <= kOrderMaxSegs &&
      nseg > g * kWarps) {
    auto *base = static_cast<unsigned char *>(d_ws);
    auto *st = reinterpret_cast<OrderState *>(base + kOrderStateOffset);
    order = reinterpret_cast<unsigned int *>(base + kOrderOffset);
    const unsigned og = static_cast<unsigned>((nseg + kOrderThreads - 1) / kOrderThreads);
    const unsigned long long tail = static_cast<unsigned long long>(EXSUM_SEG_TAIL) * g * kWarps;
    const unsigned long long tail_start = nseg > tail ? nseg - tail : 0;
    const unsigned hg =
        static_cast<unsigned>((nseg - tail_start + kOrderThreads - 1) / kOrderThreads);
    exsum_segment_hist_kernel<<<hg, kOrderThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        offs, nseg, tail_start, st);
    exsum_segment_scatter_kernel<<<og, kOrderThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        offs, nseg, tail_start, st, order);
  }
  // Deferred rounding: raw records go to d_partials when the caller wants them,
  // else to the workspace after the claim order (when it has room).
  exsum_partial *raw = nullptr;
#if EXSUM_SEG_DEFER
  if (d_partials) {
    raw = d_partials;
  } else if (order && ws_bytes >= exsum_cuda_segmented_workspace_bytes(nseg)) {
    raw = reinterpret_cast<exsum_partial *>(static_cast<unsigned char *>(d_ws) +
                                            seg_records_offset(nseg));
  }
#endif
  exsum_segmented_kernel<<<static_cast<unsigned>(g), kThreads, kSmem,
                           static_cast<cudaStream_t>(stream)>>>(
      d_x, offs, nseg, static_cast<Workspace *>(d_ws), d_out, d_partials, order, raw);
  if (raw)
    exsum_segment_emit_kernel<<<static_cast<unsigned>((nseg + kEmitWarps - 1) / kEmitWarps),
                                32 * kEmitWarps, 0, static_cast<cudaStream_t>(stream)>>>(
        raw, offs, d_x, nseg, d_out, d_partials);
  return launch_status();
}

size_t exsum_cuda_segmented_workspace_bytes(size_t nseg) {
  // never below the plain-sum workspace, so one buffer serves both kinds of call
  const size_t base = exsum_cuda_workspace_bytes();
  if (nseg > kOrderMaxSegs) return base;
#if EXSUM_SEG_DEFER
  const size_t need = seg_records_offset(nseg) + nseg * sizeof(exsum_partial);
#else
  const size_t need = kOrderOffset + 4 * nseg;
#endif
  return need > base ? need : base;
}

int exsum_cuda_merge(const exsum_partial *d_parts, size_t k, double *d_result,
                     exsum_partial *d_out, void *stream) {
  EXSUM_NVTX("exsum_cuda_merge");
  if (k && !d_parts) return EXSUM_EINVAL;
  exsum_merge_kernel<<<1, 96, 0, static_cast<cudaStream_t>(stream)>>>(d_parts, k, d_result,
                                                                      d_out);
  return launch_status();
}

#if EXSUM_TIMELINE
int exsum_debug_seg_timeline(unsigned long long *out, size_t count) {
  if (!out || count > sizeof(g_seg_timeline) / 8) return EXSUM_EINVAL;
  return cudaMemcpyFromSymbol(out, g_seg_timeline, count * 8) == cudaSuccess ? EXSUM_OK
                                                                             : EXSUM_ECUDA;
}

int exsum_debug_timeline(unsigned long long *out, size_t count) {
  if (!out || count > sizeof(g_timeline) / 8) return EXSUM_EINVAL;
  return cudaMemcpyFromSymbol(out, g_timeline, count * 8) == cudaSuccess ? EXSUM_OK : EXSUM_ECUDA;
}
#endif

}  // extern "C"
