// sum_kernels.cu — the sm_100a exact-summation hot path.
//
// Replaces exact_sum(values, ExactMethod::large) (vector_ops.cpp:121-130), i.e.
// LargeAccumulator::add(span) + drain + SmallAccumulator::round
// (large_accumulator.cpp:28-136, small_accumulator.cpp:244-348), and the
// split-merge of parallel_exact_sum (vector_ops.cpp:172-186).  See DESIGN.md.
//
// Device representation (B200-first, not the reference's): every LANE owns a
// private superaccumulator of 66 "slots" in shared memory.  Slot k holds a
// signed 96-bit integer V_k with weight 2^(32k - 1075) — the reference's chunk
// weight — stored as two planes, a u32 low word L[k][lane] and an s64 high word
// H[k][lane].  A term with biased exponent e' = max(e, 1) and signed significand
// t (53 bits with the implicit one) adds t * 2^(e' & 31) (< 2^84 in magnitude)
// to slot e' >> 5 with one 96-bit add: 3 integer instructions, 1 LDS.32 +
// 1 LDS.64 + 1 STS.32 + 1 STS.64, no atomics and no bank conflicts (lane-
// interleaved planes), independent of how the exponents are distributed.  96-bit
// slots with 2^11 headroom absorb 2047 terms; each lane renormalises (carries
// upward, leaving L in [0,2^32) and H = 0) at most every 2016 terms.
//
// Why not the reference's 4096 shared bins: 64-bit shared atomics compile to
// ATOMS.CAST.SPIN.64 CAS loops on sm_100a and random-bin read-modify-writes
// cost ~3.5x in bank conflicts; narrow data (U[0,1)) puts half of all terms in
// one bin.  Lane privatisation makes all three problems disappear.
//
// Kernels
//   exsum_sum_kernel        K1+K2+K3: persistent grid, 8 warps/CTA, each warp
//                           streams a contiguous range with 256-bit loads
//                           (double-buffered), lanes accumulate privately; the
//                           CTA combines its 8x32 lanes into 67 chunk sums,
//                           REDG.ADD.64 into the workspace; the last CTA
//                           canonicalises, resolves Inf/NaN and rounds.
//   exsum_segmented_kernel  K4: one warp per segment (dynamic), same inner loop,
//                           warp-local combine + round, one double per segment.
//   exsum_merge_kernel      K5: merge of k gathered partial records + round.

#include <cuda_runtime.h>
#include <stdint.h>

#include "exsum_b200.h"
#include "exsum_core.h"

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

// ---------------------------------------------------------- lane accumulators

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kSlots = 66;       // slots 0..63 take terms, 64..65 only carries
#ifndef EXSUM_VEC_PER_LANE
#define EXSUM_VEC_PER_LANE 8
#endif
constexpr int kVecPerLane = EXSUM_VEC_PER_LANE;  // 256-bit vectors per lane per batch
constexpr int kBatchTerms = kVecPerLane * 4;
constexpr int kNormEvery = 2016 / kBatchTerms;   // batches between renormalisations
constexpr int kLPlane = kSlots * 32 * 4;
constexpr int kHPlane = kSlots * 32 * 8;
constexpr int kWarpSmem = kLPlane + kHPlane;              // 25,344 B
constexpr int kScratch = kWarps * kChunks * 8;            // per-warp chunk rows
constexpr int kSumSmem = kWarps * kWarpSmem + kScratch;   // 207,040 B

// One lane's view of its accumulator.  Generic pointers serve the cold paths
// (renormalisation, reduction); the hot path uses 32-bit shared addresses:
// slot k's low word is at sl + 128 k and its high word at 2 * (sl + 128 k) + hoff.
struct Lane {
  uint32_t *L;                  // &Lplane[0][lane]; slot k at L[32 k]
  unsigned long long *H;        // &Hplane[0][lane]; slot k at H[32 k]
  uint32_t sl;                  // shared address of L[0][lane]
  uint32_t hoff;                // shared address of H[0][lane] minus 2 * sl
};

struct Specials {                // first occurrences seen by one lane
  unsigned long long P, M, N;    // index (global or segment-local), ~0 = none
};

__device__ __forceinline__ Lane lane_view(unsigned char *warp_smem, int lane) {
  Lane v;
  v.L = reinterpret_cast<uint32_t *>(warp_smem) + lane;
  v.H = reinterpret_cast<unsigned long long *>(warp_smem + kLPlane) + lane;
  v.sl = static_cast<uint32_t>(__cvta_generic_to_shared(v.L));
  v.hoff = static_cast<uint32_t>(__cvta_generic_to_shared(v.H)) - 2u * v.sl;
  return v;
}

// Zero one warp's planes cooperatively with 16-byte stores.
__device__ __forceinline__ void zero_warp_planes(unsigned char *warp_smem, int lane) {
  uint4 *p = reinterpret_cast<uint4 *>(warp_smem);
  constexpr int n16 = kWarpSmem / 16;
#pragma unroll 4
  for (int i = lane; i < n16; i += 32) p[i] = make_uint4(0, 0, 0, 0);
}

__device__ __forceinline__ uint32_t exponent_field(uint32_t hi) { return (hi >> 20) & 0x7FFu; }

// Add one finite term (exponent field e != 2047, e passed in) to the lane's slots.
//
// The term is (-1)^s * m * 2^(e' - 1075), e' = max(e, 1), m the significand with
// its implicit one.  In slot units it is m << (e' & 31) added at slot e' >> 5;
// m << sh spans 96 bits (u2:u1:u0).  Negative terms add ~(m << sh) + 1: the
// complement is folded into the funnel shifts (fill words = s) and the +1 is
// the carry-in of the 96-bit add (CC.CF = s & 1 from s + s).  -0.0 adds 2^96,
// i.e. nothing.  ~23 SASS per term: no branches, no atomics.
__device__ __forceinline__ void add_term(const Lane &a, uint32_t lo, uint32_t hi, uint32_t e) {
  const uint32_t ep = max(e, 1u);                          // denormal: exponent 1
  const uint32_t imp = e ? 0x100000u : 0u;                  // implicit one
  const uint32_t s = static_cast<uint32_t>(static_cast<int32_t>(hi) >> 31);
  const uint32_t mx = ((hi & 0xFFFFFu) | imp) ^ s;
  const uint32_t lx = lo ^ s;
  const uint32_t u0 = __funnelshift_l(s, lx, ep);         // shift count taken mod 32
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
    add_term(a, lo, hi, e);
  }
}

// Carry upward through the lane's slots: afterwards L_k in [0, 2^32), H_k = 0
// for k < 65 and slot 65 holds the rest.  Safe whenever every slot has seen at
// most 2047 terms since the last call (|H_k| < 2^63 - 2^52).
__device__ __forceinline__ void normalize_lane(const Lane &a) {
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

// Warp-wide sum of the 32 normalised lane accumulators into chunk values.
// Lane j returns rows j, j+32 and (j < 2) j+64 in r0, r1, r2; every lane returns
// chunk 66 (the sum of the slot-65 high words) in r66.  Reads are skewed so the
// 32 lanes hit 32 distinct banks.
__device__ __forceinline__ void warp_reduce_planes(unsigned char *warp_smem, int lane,
                                                   long long &r0, long long &r1,
                                                   long long &r2, long long &r66) {
  const uint32_t *Lp = reinterpret_cast<const uint32_t *>(warp_smem);
  const unsigned long long *Hp = reinterpret_cast<const unsigned long long *>(warp_smem + kLPlane);
  unsigned long long s0 = 0, s1 = 0, s2 = 0;
  const int rowa = lane, rowb = lane + 32, rowc = lane + 64;
#pragma unroll 8
  for (int i = 0; i < 32; ++i) {
    const int col = (i + lane) & 31;
    s0 += Lp[rowa * 32 + col];
    s1 += Lp[rowb * 32 + col];
    if (rowc < kSlots) s2 += Lp[rowc * 32 + col];
  }
  long long h = static_cast<long long>(Hp[(kSlots - 1) * 32 + lane]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  r0 = static_cast<long long>(s0);
  r1 = static_cast<long long>(s1);
  r2 = static_cast<long long>(s2);
  r66 = h;
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

// Process one batch (kBatchTerms terms per lane).  index_of_vec0 is the
// special-value index of term 0 of vector v0 of the batch.
__device__ __forceinline__ void process_batch(const Lane &a, Specials &sp, Batch &b, int lane,
                                              unsigned long long index_of_vec0) {
  uint32_t e[kVecPerLane][4];
  bool special = false;
#pragma unroll
  for (int u = 0; u < kVecPerLane; ++u)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      e[u][q] = exponent_field(b.w[u][2 * q + 1]);
      special |= e[u][q] == 0x7FFu;
    }
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
#pragma unroll
  for (int u = 0; u < kVecPerLane; ++u)
#pragma unroll
    for (int q = 0; q < 4; ++q) add_term(a, b.w[u][2 * q], b.w[u][2 * q + 1], e[u][q]);
}

// Accumulate x[begin, end) into the calling warp's lane slots.  `index_base`
// is added to positions to form special-value indices.  norm_count tracks
// batches since the last renormalisation (warp-uniform).
__device__ void warp_accumulate(const double *__restrict__ x, unsigned long long begin,
                                unsigned long long end, unsigned long long index_base,
                                const Lane &a, Specials &sp, int &norm_count, int lane) {
  if (begin >= end) return;
  // Scalar head up to 32-byte alignment of &x[pos].
  const uintptr_t addr = reinterpret_cast<uintptr_t>(x + begin);
  unsigned long long head = ((32u - (addr & 31u)) & 31u) >> 3;
  if (head > end - begin) head = end - begin;
  if (lane < static_cast<int>(head)) {
    const unsigned long long bits = __ldg(reinterpret_cast<const unsigned long long *>(x) + begin + lane);
    add_term_checked(a, sp, static_cast<uint32_t>(bits), static_cast<uint32_t>(bits >> 32),
                     index_base + begin + lane);
  }
  const unsigned long long vbeg_t = begin + head;  // first vector's term position
  const long long nvec = static_cast<long long>((end - vbeg_t) >> 2);
  const double *X4 = x + vbeg_t;                   // 32-byte aligned
  const unsigned long long tail_t = vbeg_t + 4ull * static_cast<unsigned long long>(nvec);
  if (lane < static_cast<int>(end - tail_t)) {
    const unsigned long long bits = __ldg(reinterpret_cast<const unsigned long long *>(x) + tail_t + lane);
    add_term_checked(a, sp, static_cast<uint32_t>(bits), static_cast<uint32_t>(bits >> 32),
                     index_base + tail_t + lane);
  }
  if (nvec <= 0) return;
  constexpr long long kStep = kVecPerLane * 32;
  Batch b0, b1;
  long long v = 0;
  load_batch(b0, X4, 0, nvec, lane);
  const unsigned long long ib = index_base + vbeg_t;
  while (true) {
    long long nx = v + kStep;
    if (nx < nvec) load_batch(b1, X4, nx, nvec, lane);
    process_batch(a, sp, b0, lane, ib + 4ull * static_cast<unsigned long long>(v));
    if (++norm_count >= kNormEvery) {
      normalize_lane(a);
      norm_count = 0;
    }
    v = nx;
    if (v >= nvec) break;
    nx = v + kStep;
    if (nx < nvec) load_batch(b0, X4, nx, nvec, lane);
    process_batch(a, sp, b1, lane, ib + 4ull * static_cast<unsigned long long>(v));
    if (++norm_count >= kNormEvery) {
      normalize_lane(a);
      norm_count = 0;
    }
    v = nx;
    if (v >= nvec) break;
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

// Finalise a canonical record: resolve specials, round, write outputs.
__device__ void emit_record(int64_t *c, unsigned long long P, unsigned long long M,
                            unsigned long long N, unsigned long long payload, double *result,
                            exsum_partial *partial) {
  const int top = exsum_canonicalize(c);
  uint64_t ib, nb;
  exsum_resolve_specials(P, M, N, payload, &ib, &nb);
  if (result) *result = __longlong_as_double(static_cast<long long>(exsum_result_bits(ib, nb, c, top)));
  if (partial) {
    for (int i = 0; i < kChunks; ++i) partial->acc.chunk[i] = c[i];
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

// --------------------------------------------------------------- K1 + K2 + K3

__global__ void __launch_bounds__(kThreads, 1)
exsum_sum_kernel(const double *__restrict__ x, unsigned long long n,
                 unsigned long long base_index, Workspace *__restrict__ ws, int finalize,
                 double *result, exsum_partial *partial) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char *wsm = smem + warp * kWarpSmem;
  long long *scratch = reinterpret_cast<long long *>(smem + kWarps * kWarpSmem);
  zero_warp_planes(wsm, lane);
  __syncwarp();
  const Lane a = lane_view(wsm, lane);
  Specials sp{~0ull, ~0ull, ~0ull};
  int norm_count = 0;

  // Contiguous per-warp ranges, boundaries on 4-term multiples.
  const unsigned long long gw = static_cast<unsigned long long>(blockIdx.x) * kWarps + warp;
  const unsigned long long nw = static_cast<unsigned long long>(gridDim.x) * kWarps;
  const unsigned long long quads = (n + 3) >> 2;
  const unsigned long long qb = quads * gw / nw, qe = quads * (gw + 1) / nw;
  const unsigned long long tb = qb * 4, te = min(qe * 4, n);
  warp_accumulate(x, tb, te, base_index, a, sp, norm_count, lane);

  // K2: lane renormalisation and the warp's 67 chunk sums.
  normalize_lane(a);
  __syncwarp();
  long long r0, r1, r2, r66;
  warp_reduce_planes(wsm, lane, r0, r1, r2, r66);
  long long *row = scratch + warp * kChunks;
  row[lane] = r0;
  row[lane + 32] = r1;
  if (lane < 2) row[lane + 64] = r2;
  if (lane == 0) row[66] = r66;
  const unsigned long long P = warp_min_u64(sp.P), M = warp_min_u64(sp.M),
                           N = warp_min_u64(sp.N);
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
  __threadfence();
  if (threadIdx.x != 0) return;
  // Last CTA: the NaN payload of the first NaN, if it lies in this launch.
  const unsigned long long Nf = ~__ldcg(&ws->inv_nan);
  unsigned long long payload = __ldcg(&ws->nan_payload);
  if (Nf != ~0ull && Nf >= base_index && Nf - base_index < n) {
    payload = __ldcg(reinterpret_cast<const unsigned long long *>(x) + (Nf - base_index));
    ws->nan_payload = payload;
  }
  ws->done = 0;
  if (!finalize) return;
  int64_t c[kChunks];
  for (int i = 0; i < kChunks; ++i) {
    c[i] = static_cast<int64_t>(__ldcg(&ws->chunk[i]));
    ws->chunk[i] = 0;
  }
  const unsigned long long Pf = ~__ldcg(&ws->inv_pinf), Mf = ~__ldcg(&ws->inv_ninf);
  ws->inv_pinf = ws->inv_ninf = ws->inv_nan = 0;
  ws->nan_payload = 0;
  emit_record(c, Pf, Mf, Nf, payload, result, partial);
}

// Finalise a workspace filled by exsum_cuda_accumulate launches.
__global__ void exsum_finalize_kernel(Workspace *ws, double *result, exsum_partial *partial) {
  int64_t c[kChunks];
  for (int i = 0; i < kChunks; ++i) {
    c[i] = static_cast<int64_t>(ws->chunk[i]);
    ws->chunk[i] = 0;
  }
  const unsigned long long P = ~ws->inv_pinf, M = ~ws->inv_ninf, N = ~ws->inv_nan;
  const unsigned long long payload = ws->nan_payload;
  ws->inv_pinf = ws->inv_ninf = ws->inv_nan = 0;
  ws->nan_payload = 0;
  ws->done = 0;
  emit_record(c, P, M, N, payload, result, partial);
}

// ------------------------------------------------------------------------- K4

constexpr int kSegSmem = kWarps * kWarpSmem + kScratch;

__global__ void __launch_bounds__(kThreads, 1)
exsum_segmented_kernel(const double *__restrict__ x, const unsigned long long *__restrict__ offs,
                       unsigned long long nseg, Workspace *__restrict__ ws, double *out,
                       exsum_partial *partials) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char *wsm = smem + warp * kWarpSmem;
  long long *row = reinterpret_cast<long long *>(smem + kWarps * kWarpSmem) + warp * kChunks;
  const Lane a = lane_view(wsm, lane);
  while (true) {
    unsigned int s = 0;
    if (lane == 0) s = atomicAdd(&ws->seg_next, 1u);
    s = __shfl_sync(0xffffffffu, s, 0);
    if (s >= nseg) break;
    zero_warp_planes(wsm, lane);
    __syncwarp();
    const unsigned long long b = offs[s], e = offs[s + 1];
    Specials sp{~0ull, ~0ull, ~0ull};
    int norm_count = 0;
    // indices local to the segment: position - b
    warp_accumulate(x, b, e, 0ull - b, a, sp, norm_count, lane);
    normalize_lane(a);
    __syncwarp();
    long long r0, r1, r2, r66;
    warp_reduce_planes(wsm, lane, r0, r1, r2, r66);
    row[lane] = r0;
    row[lane + 32] = r1;
    if (lane < 2) row[lane + 64] = r2;
    if (lane == 0) row[66] = r66;
    const unsigned long long P = warp_min_u64(sp.P), M = warp_min_u64(sp.M),
                             N = warp_min_u64(sp.N);
    __syncwarp();
    if (lane == 0) {
      int64_t c[kChunks];
      for (int i = 0; i < kChunks; ++i) c[i] = row[i];
      const unsigned long long payload =
          N != ~0ull ? __ldg(reinterpret_cast<const unsigned long long *>(x) + b + N) : 0ull;
      emit_record(c, P, M, N, payload, out + s, partials ? partials + s : nullptr);
    }
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
  if (t == 0) {
    int64_t c[kChunks];
    for (int i = 0; i < kChunks; ++i) c[i] = sc[i];
    emit_record(c, sP, sM, sN, sPay, result, out);
  }
}

}  // namespace dev
}  // namespace exsum_b200

// ===================================================================== C ABI

using namespace exsum_b200;
using namespace exsum_b200::dev;

namespace {

int g_num_sms = 0;

int num_sms() {
  if (g_num_sms > 0) return g_num_sms;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  g_num_sms = sms;
  return sms;
}

bool configured = false;

int configure_kernels() {
  if (configured) return EXSUM_OK;
  if (cudaFuncSetAttribute(exsum_sum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSumSmem) != cudaSuccess)
    return EXSUM_ECUDA;
  if (cudaFuncSetAttribute(exsum_segmented_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSegSmem) != cudaSuccess)
    return EXSUM_ECUDA;
  configured = true;
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
               void *stream, int finalize, double *d_result, exsum_partial *d_partial) {
  if (!d_ws || ws_bytes < sizeof(Workspace) || (n && !d_x)) return EXSUM_EINVAL;
  int st = configure_kernels();
  if (st) return st;
  const int sms = num_sms();
  if (sms <= 0) return EXSUM_ECUDA;
  const unsigned grid = grid_for(n, sms);
  exsum_sum_kernel<<<grid, kThreads, kSumSmem, static_cast<cudaStream_t>(stream)>>>(
      d_x, n, base_index, static_cast<Workspace *>(d_ws), finalize, d_result, d_partial);
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

int exsum_cuda_accumulate(const double *d_x, size_t n, uint64_t base_index, void *d_ws,
                          size_t ws_bytes, void *stream) {
  if (n == 0) return (d_ws && ws_bytes >= sizeof(Workspace)) ? EXSUM_OK : EXSUM_EINVAL;
  return sum_launch(d_x, n, base_index, d_ws, ws_bytes, stream, 0, nullptr, nullptr);
}

int exsum_cuda_finalize(double *d_result, exsum_partial *d_partial, void *d_ws, size_t ws_bytes,
                        void *stream) {
  if (!d_ws || ws_bytes < sizeof(Workspace)) return EXSUM_EINVAL;
  exsum_finalize_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
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
  int st = configure_kernels();
  if (st) return st;
  const int sms = num_sms();
  if (sms <= 0) return EXSUM_ECUDA;
  unsigned long long g = (nseg + kWarps - 1) / kWarps;
  if (g > static_cast<unsigned long long>(sms)) g = sms;
  exsum_segmented_kernel<<<static_cast<unsigned>(g), kThreads, kSegSmem,
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
