// Probe: the north_star's suggested per-term step, measured as an UPPER BOUND
// of that design (no per-bin counts, no 4096-add transfers, no drain), against
// the lane-private 96-bit accumulators this repo uses.
//
// Every variant streams n float64 terms (LDG.128, grid-stride, 4 loads in
// flight per thread) and adds each term's raw 64-bit pattern to the bin of its
// 12 sign+exponent bits, as LargeAccumulator::add does (large_accumulator.hpp:
// 47-59: chunks[bits >> 52] += bits):
//   atom64      4096 u64 bins per CTA in shared memory, atomicAdd per term
//               (sm_100a: ATOMS.CAST.SPIN.64, a CAS loop)
//   match64     __match_any_sync on the bin index, the group's patterns summed
//               with three __reduce_add_sync of 22-bit pieces, one CAS-loop
//               atomicAdd per group (the north_star's warp pre-combining)
//   warpbins    4096 u64 bins per WARP (32 KB; 6 warps per SM), match_any +
//               reductions, the group leader does a plain LDS.64/STS.64 update
//               (no atomics: the warp owns its bins)
// Data (seeded SplitMix64 of the index): c2 = U[0,1) (half the terms in one
// bin), c3 = random sign/exponent 1..2046/mantissa + 1% denormals, c4 = ±10^u,
// u ~ U[-20, 20] (about 270 bins).  Prints GB/s (8 bytes per term) per variant.
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gen(double *x, uint64_t n, int config) {
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t r = splitmix(i * 7919u + config), r2 = splitmix(r);
    double v;
    if (config == 2) {
      v = (r >> 11) * 0x1.0p-53;
    } else if (config == 3) {
      const uint64_t e = (r2 % 100 == 0) ? 0 : 1 + (r2 >> 8) % 2046;
      v = __longlong_as_double((r & 0x800FFFFFFFFFFFFFull) | (e << 52));
    } else {
      const double u = ((r >> 11) * 0x1.0p-53) * 40.0 - 20.0;
      v = exp10(u) * ((r2 & 1) ? -1.0 : 1.0);
    }
    x[i] = v;
  }
}

constexpr int kBins = 4096;

template <int KIND>
__device__ __forceinline__ void add_bits(unsigned long long *bins, unsigned long long bits) {
  const unsigned ix = static_cast<unsigned>(bits >> 52);
  if (KIND == 0) {
    atomicAdd(bins + ix, bits);
  } else {
    const unsigned m = __match_any_sync(0xffffffffu, ix);
    const unsigned p0 = __reduce_add_sync(m, static_cast<unsigned>(bits & 0x3FFFFF));
    const unsigned p1 = __reduce_add_sync(m, static_cast<unsigned>((bits >> 22) & 0x3FFFFF));
    const unsigned p2 = __reduce_add_sync(m, static_cast<unsigned>(bits >> 44));
    if ((__ffs(m) - 1) == static_cast<int>(threadIdx.x & 31)) {
      const unsigned long long s = p0 + (static_cast<unsigned long long>(p1) << 22) +
                                   (static_cast<unsigned long long>(p2) << 44);
      if (KIND == 1) {
        atomicAdd(bins + ix, s);
      } else {
        bins[ix] += s;  // warp-private bins: plain read-modify-write
      }
    }
  }
}

template <int KIND, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) bins_kernel(const double *x, uint64_t n,
                                                          unsigned long long *out) {
  extern __shared__ unsigned long long sb[];
  const int warp = threadIdx.x >> 5;
  unsigned long long *bins = KIND == 2 ? sb + warp * kBins : sb;
  const int nb = KIND == 2 ? WARPS * kBins : kBins;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) sb[i] = 0;
  __syncthreads();
  const uint64_t n2 = n / 2;  // 16-byte pairs
  const ulonglong2 *x2 = reinterpret_cast<const ulonglong2 *>(x);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {  // warp-uniform trip count (n2 % stride == 0 below)
    ulonglong2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(x2 + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      add_bits<KIND>(bins, v[u].x);
      add_bits<KIND>(bins, v[u].y);
    }
  }
  for (; i < n2; i += stride) {
    const ulonglong2 v = __ldcs(x2 + i);
    add_bits<KIND>(bins, v.x);
    add_bits<KIND>(bins, v.y);
  }
  __syncthreads();
  unsigned long long acc = 0;
  for (int k = threadIdx.x; k < nb; k += blockDim.x) acc += sb[k];
  atomicAdd(out, acc);  // keeps the work observable
}

template <int KIND, int WARPS>
float run(const double *x, uint64_t n, unsigned long long *out, int sms) {
  auto k = bins_kernel<KIND, WARPS>;
  const int smem = (KIND == 2 ? WARPS : 1) * kBins * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, WARPS * 32, smem);
  const int grid = sms * per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k<<<grid, WARPS * 32, smem>>>(x, n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t n = 100000000ull / (2ull * 148 * 1024) * (2ull * 148 * 1024);  // ~1e8, whole strides
  double *x;
  unsigned long long *out;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&out, 8);
  printf("n = %llu terms (%d SMs); GB/s = 8 bytes per term / best of 3\n",
         static_cast<unsigned long long>(n), sms);
  for (int config : {2, 3, 4}) {
    gen<<<sms * 8, 256>>>(x, n, config);
    cudaDeviceSynchronize();
    const float a = run<0, 32>(x, n, out, sms);   // 1024 threads, 32 KB bins per CTA
    const float b = run<1, 32>(x, n, out, sms);
    const float c = run<2, 6>(x, n, out, sms);    // 6 warps x 32 KB
    printf("config %d: atom64 %.3f ms %.0f GB/s | match64 %.3f ms %.0f GB/s | warpbins %.3f ms %.0f GB/s\n",
           config, a, 8.0 * n / a / 1e6, b, 8.0 * n / b / 1e6, c, 8.0 * n / c / 1e6);
  }
  return 0;
}
