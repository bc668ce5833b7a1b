// host_tools.cpp — the paper's benchmark data generator behind the C ABI
// (formats and tooling).
//
// generate() (generator.cpp:23-45, generator.hpp:24-58): n/2 values
// U1 * exp(30 U2) from a minstd multiplicative congruential stream
// (x <- 48271 x mod 2^31 - 1, uniform on (0,1) as x / (2^31 - 1)), mirrored
// as -v into the second half so the exact sum is zero; optionally a
// Fisher-Yates shuffle driven by the same stream.  The paper's timing data
// and a zero-sum known answer for every exact method.

#include <cmath>
#include <cstdint>
#include <utility>

#include "exsum_b200.h"

namespace {

struct Minstd {
  static constexpr uint64_t kA = 48271, kM = (uint64_t{1} << 31) - 1;
  uint64_t x;
  explicit Minstd(uint64_t seed) : x(seed % (kM - 1) + 1) {}
  uint32_t next() {
    x = (kA * x) % kM;  // < 2^47: exact in 64 bits
    return static_cast<uint32_t>(x);
  }
  double unit() { return static_cast<double>(next()) / static_cast<double>(kM); }
};

}  // namespace

extern "C" int exsum_generate(uint64_t n, uint64_t seed, int permute, double *out) {
  if (n == 0 || n % 2 != 0 || !out) return EXSUM_EINVAL;
  Minstd rng(seed);
  const uint64_t half = n / 2;
  for (uint64_t i = 0; i < half; ++i) {
    const double u1 = rng.unit();
    const double u2 = rng.unit();
    out[i] = u1 * std::exp(30.0 * u2);
    out[n - 1 - i] = -out[i];
  }
  if (permute) {
    for (uint64_t i = n - 1; i > 0; --i) {
      const uint64_t j = rng.next() % (i + 1);
      std::swap(out[i], out[j]);
    }
  }
  return EXSUM_OK;
}
