// Pipe-assignment / throughput probe for integer instruction forms on sm_100a.
// Each kernel: 8 independent chains, each step = probe op followed by an xor with a
// per-chain register (LOP3), so ptxas cannot fold the chain.  Run under
// `ncu --metrics sm__inst_executed_pipe_{alu,fma,fmaheavy,fmalite}.sum` to see
// which pipe executes the probe op; wall time gives throughput.
#include <cstdint>
#include <cstdio>
#define ITER 2048
#define CH 8
#define K(NAME, BODY)                                                                    \
  __global__ void NAME(uint32_t *out, uint32_t a0, uint32_t b0) {                        \
    uint32_t r[CH], m[CH];                                                               \
    for (int c = 0; c < CH; ++c) {                                                       \
      r[c] = threadIdx.x * 7u + c + a0;                                                  \
      m[c] = b0 * (c + 3) + threadIdx.x;                                                 \
    }                                                                                    \
    uint32_t b = b0 + threadIdx.x;                                                       \
    _Pragma("unroll 8") for (int i = 0; i < ITER; ++i) {                                 \
      _Pragma("unroll") for (int c = 0; c < CH; ++c) {                                   \
        uint32_t x = r[c];                                                               \
        BODY;                                                                            \
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(x) : "r"(m[c]));                       \
        r[c] = x;                                                                        \
      }                                                                                  \
    }                                                                                    \
    uint32_t s = 0;                                                                      \
    for (int c = 0; c < CH; ++c) s ^= r[c];                                              \
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;                                      \
  }
K(k_base, (void)b)
K(k_iadd, asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(b)))
K(k_viadd, asm volatile("add.u32 %0, %0, 0x1357;" : "+r"(x)))
K(k_shf, asm volatile("shf.l.wrap.b32 %0, %0, %1, %0;" : "+r"(x) : "r"(b)))
K(k_shr, asm volatile("shr.u32 %0, %0, 3;" : "+r"(x)))
K(k_imad, asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(x) : "r"(b)))
K(k_imadhi, asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x) : "r"(b)))
K(k_min, asm volatile("min.u32 %0, %0, %1;" : "+r"(x) : "r"(b)))
K(k_selp, asm volatile("{.reg .pred p; setp.ne.u32 p, %0, %1; selp.u32 %0, %0, %1, p;}"
                       : "+r"(x)
                       : "r"(b)))
K(k_prmt, asm volatile("prmt.b32 %0, %0, %1, 0x1032;" : "+r"(x) : "r"(b)))
K(k_lea, asm volatile("{.reg .u32 t; shl.b32 t, %0, 4; add.u32 %0, t, %1;}" : "+r"(x) : "r"(b)))
K(k_isetp, asm volatile("{.reg .pred p; setp.lt.u32 p, %0, %1; @p add.u32 %0, %0, 1;}"
                        : "+r"(x)
                        : "r"(b)))

int main() {
  uint32_t *out;
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  struct {
    const char *n;
    void (*f)(uint32_t *, uint32_t, uint32_t);
  } ks[] = {{"base", k_base}, {"iadd", k_iadd},     {"viadd", k_viadd}, {"shf", k_shf},
            {"shr", k_shr},   {"imad", k_imad},     {"imadhi", k_imadhi}, {"min", k_min},
            {"selp", k_selp}, {"prmt", k_prmt},     {"lea", k_lea},     {"isetp", k_isetp}};
  for (auto &k : ks) {
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(s);
      k.f<<<148 * 8, 256>>>(out, 1, 3);
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      cudaEventElapsedTime(&ms, s, e);
    }
    double steps = 148.0 * 8 * 256 * ITER * CH;
    printf("%-8s %8.3f ms  %6.1f steps/clk/SM (@1.9GHz)\n", k.n, ms,
           steps / (ms * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
