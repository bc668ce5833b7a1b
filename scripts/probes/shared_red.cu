// Shared-memory update probe (sm_100a): cost of one lane-private accumulator
// update per lane per step, 8 warps x 148 CTAs, lane-interleaved addresses
// (conflict-free), slot chosen per step by a cheap hash (all lanes differ).
//   rmw96: LDS + LDS.64, 96-bit add, STS + STS.64     (the current design)
//   red5:  5 x red.shared.add.u32 on consecutive digit rows (a 16-bit digit design)
//   red4:  4 x red.shared.add.u32
//   red64: 2 x red.shared.add.u64 (CAS loop on sm_100a?)
//   sts5:  5 x st.shared.u32 (store-only reference)
//   rmw96+ldg / rmw3x32+ldg / rmw96+ldgNA: the RMW (as u32 + u64 or as three
//          u32 planes) with a concurrent 32-byte streaming load per lane
//          (L1::evict_first or L1::no_allocate): shared-store bank conflicts
//          appear only with the global stream?
// Wall time (CUDA events) per step per SM; run under ncu for wavefronts.
#include <cstdint>
#include <cstdio>
#define STEPS 4096
#define WARPS 8
#define ROWS 192  // u32 rows per lane (24 KB per warp), lane-interleaved: row r of lane l at [r*32 + l]

template <int KIND>
__global__ void __launch_bounds__(WARPS * 32, 1) probe(uint32_t *out, uint32_t seed,
                                                       const uint4 *g) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t *w = sm + warp * ROWS * 32;
  for (int i = lane; i < ROWS * 32; i += 32) w[i] = 0;
  __syncwarp();
  uint32_t h = seed ^ (threadIdx.x * 0x9E3779B9u), v = h | 1u;
  const uint32_t wbase = static_cast<uint32_t>(__cvta_generic_to_shared(w));
  const uint32_t base = wbase + 4u * lane;           // u32 rows
  const uint32_t hbase = wbase + 8192u + 8u * lane;  // u64 rows (256 B each)
#pragma unroll 4
  for (int i = 0; i < STEPS; ++i) {
    h = h * 1664525u + 1013904223u;
    const uint32_t k = (h >> 26) & 63u;  // slot 0..63
    if (KIND == 0) {
      const uint32_t la = base + k * 128u, ha = hbase + k * 256u;
      asm volatile(
          "{.reg .u32 l, h0, h1;\n\t"
          "ld.shared.u32 l, [%0];\n\tld.shared.v2.u32 {h0, h1}, [%1];\n\t"
          "add.cc.u32 l, l, %2;\n\taddc.cc.u32 h0, h0, %2;\n\taddc.u32 h1, h1, 0;\n\t"
          "st.shared.u32 [%0], l;\n\tst.shared.v2.u32 [%1], {h0, h1};}" ::"r"(la),
          "r"(ha), "r"(v)
          : "memory");
    } else if (KIND == 1 || KIND == 2) {
      const uint32_t a = base + k * 2u * 128u;
#pragma unroll
      for (int d = 0; d < (KIND == 1 ? 5 : 4); ++d)
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a + d * 128u), "r"(v + d) : "memory");
    } else if (KIND == 3) {
      const uint32_t a = base + k * 128u;  // u64 rows: two rows per slot at 256 B stride
      asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(hbase + (k & 15u) * 512u), "l"((unsigned long long)v) : "memory");
      asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(hbase + (k & 15u) * 512u + 256u), "l"((unsigned long long)v) : "memory");
      (void)a;
    } else if (KIND == 4) {
      const uint32_t a = base + k * 2u * 128u;
#pragma unroll
      for (int d = 0; d < 5; ++d)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a + d * 128u), "r"(v + d) : "memory");
    } else {
      // KIND 5: rmw96 + a 32-byte streaming load per lane per step; KIND 6: the
      // same RMW as three u32 planes (L, H0, H1) + the load; KIND 7: rmw96 + load
      // through L1::no_allocate
      uint32_t w[8];
      const uint4 *src = g + 2 * ((static_cast<size_t>(blockIdx.x) * WARPS * 32 + threadIdx.x) +
                                  static_cast<size_t>(i) * 148 * WARPS * 32);
      if (KIND == 7)
        asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                       "=r"(w[6]), "=r"(w[7]) : "l"(src));
      else
        asm volatile("ld.global.nc.L1::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                       "=r"(w[6]), "=r"(w[7]) : "l"(src));
      const uint32_t x = w[0] ^ w[1] ^ w[2] ^ w[3] ^ w[4] ^ w[5] ^ w[6] ^ w[7];
      if (KIND == 6) {
        const uint32_t la = base + k * 128u, h0 = base + 64u * 128u + k * 128u,
                       h1 = base + 128u * 128u + k * 128u;
        asm volatile(
            "{.reg .u32 l, a, b;\n\t"
            "ld.shared.u32 l, [%0];\n\tld.shared.u32 a, [%1];\n\tld.shared.u32 b, [%2];\n\t"
            "add.cc.u32 l, l, %3;\n\taddc.cc.u32 a, a, %3;\n\taddc.u32 b, b, 0;\n\t"
            "st.shared.u32 [%0], l;\n\tst.shared.u32 [%1], a;\n\tst.shared.u32 [%2], b;}" ::"r"(la),
            "r"(h0), "r"(h1), "r"(v ^ x)
            : "memory");
      } else {
        const uint32_t la = base + k * 128u, ha = hbase + k * 256u;
        asm volatile(
            "{.reg .u32 l, h0, h1;\n\t"
            "ld.shared.u32 l, [%0];\n\tld.shared.v2.u32 {h0, h1}, [%1];\n\t"
            "add.cc.u32 l, l, %2;\n\taddc.cc.u32 h0, h0, %2;\n\taddc.u32 h1, h1, 0;\n\t"
            "st.shared.u32 [%0], l;\n\tst.shared.v2.u32 [%1], {h0, h1};}" ::"r"(la),
            "r"(ha), "r"(v ^ x)
            : "memory");
      }
    }
    v += h;
  }
  __syncwarp();
  uint32_t s = 0;
  for (int i = lane; i < ROWS * 32; i += 32) s += w[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  uint32_t *out;
  cudaMalloc(&out, 148 * WARPS * 32 * 4);
  const int smem = WARPS * ROWS * 32 * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char *names[] = {"rmw96", "red5", "red4", "red64x2", "sts5", "rmw96+ldg", "rmw3x32+ldg",
                         "rmw96+ldgNA"};
  void (*ks[])(uint32_t *, uint32_t, const uint4 *) = {probe<0>, probe<1>, probe<2>, probe<3>,
                                                       probe<4>, probe<5>, probe<6>, probe<7>};
  uint4 *g;  // 32 B per lane per step
  cudaMalloc(&g, static_cast<size_t>(148) * WARPS * 32 * STEPS * 32);
  cudaMemset(g, 1, static_cast<size_t>(148) * WARPS * 32 * STEPS * 32);
  for (int k = 0; k < 8; ++k) {
    cudaFuncSetAttribute(ks[k], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      ks[k]<<<148, WARPS * 32, smem>>>(out, 12345u + rep, g);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2)
        printf("%-8s %.3f ms  %.2f ns/step/warp  %.3f warp-steps/clk/SM (at 1.9 GHz)  err=%s\n",
               names[k], ms, ms * 1e6 / STEPS,
               (double)WARPS * STEPS / (ms * 1e-3 * 1.9e9), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
