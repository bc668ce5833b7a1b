// A C++ caller of libexsum_b200 through the C ABI only (include/exsum_b200.h):
// what a maintainer of the reference (C++20) links against.  Built and run by
// tests/test_capi.py (host part) and tests/test_gpu.py (--device part).
//
//   g++ -std=c++17 -Iinclude tests/cpp/capi_demo.cpp -Lpaper_1505_05571_b200/lib
//       -lexsum_b200 -Wl,-rpath,<that dir> -o capi_demo
//
// Prints one line per check and exits non-zero on the first mismatch.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "exsum_b200.h"

static uint64_t bits(double v) {
  uint64_t b;
  std::memcpy(&b, &v, 8);
  return b;
}

#define CHECK(cond)                                              \
  do {                                                           \
    if (!(cond)) {                                               \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      return 1;                                                  \
    }                                                            \
  } while (0)

static int host_checks() {
  // SmallAccumulator: init / add_array / round
  exsum_small acc;
  double out = -1;
  CHECK(exsum_small_init(&acc) == EXSUM_OK);
  const double v[3] = {1e15, -1e15, 0.1};
  CHECK(exsum_small_add_array(&acc, v, 3) == EXSUM_OK);
  CHECK(exsum_small_round(&acc, &out) == EXSUM_OK && out == 0.1);
  // 560-byte POD, the layout of exsum::SmallAccumulator
  static_assert(sizeof(exsum_small) == 560, "exsum_small layout");
  // LargeAccumulator: 4097 ones, counts
  exsum_large *L = exsum_large_new();
  CHECK(L != nullptr);
  std::vector<double> ones(4097, 1.0);
  CHECK(exsum_large_add_array(L, ones.data(), ones.size()) == EXSUM_OK);
  CHECK(exsum_large_round(L, &out) == EXSUM_OK && out == 4097.0);
  exsum_large_free(L);
  L = exsum_large_new();
  int count = 0;
  CHECK(exsum_large_add(L, 1.0) == EXSUM_OK);
  CHECK(exsum_large_count(L, 0x3FF, &count) == EXSUM_OK && count == 4095);
  exsum_large_free(L);
  // [1e16, 1, -1e16] -> 1, split into two partial records and merged
  const double w[3] = {1e16, 1.0, -1e16};
  exsum_partial parts[2], merged;
  CHECK(exsum_partial_from_array(w, 2, 0, &parts[0]) == EXSUM_OK);
  CHECK(exsum_partial_from_array(w + 2, 1, 2, &parts[1]) == EXSUM_OK);
  CHECK(exsum_partial_merge(parts, 2, &merged, &out) == EXSUM_OK && out == 1.0);
  // errors are status codes, not exceptions (mean of nothing, dot length mismatch)
  CHECK(exsum_small_mean(&acc, 0, &out) == EXSUM_EINVAL);
  CHECK(exsum_dot(v, 3, w, 2, &out) == EXSUM_EINVAL);
  // NaN payload survives (small_accumulator.cpp:331-333)
  uint64_t nanb = 0x7FF0000000000123ull;
  double nan_v;
  std::memcpy(&nan_v, &nanb, 8);
  const double z[3] = {1.0, nan_v, INFINITY};
  CHECK(exsum_small_init(&acc) == EXSUM_OK);
  CHECK(exsum_small_add_array(&acc, z, 3) == EXSUM_OK);
  CHECK(exsum_small_round(&acc, &out) == EXSUM_OK && bits(out) == 0x7FF0000000000123ull);
  // the library's multithreaded host kernel and the paper's generator (zero sum)
  std::vector<double> g(200'000);
  CHECK(exsum_generate(g.size(), 5, 1, g.data()) == EXSUM_OK);
  CHECK(exsum_generate(3, 5, 0, g.data()) == EXSUM_EINVAL);
  CHECK(exsum_host_sum(g.data(), g.size(), 0, 4, &out, nullptr) == EXSUM_OK && bits(out) == 0);
  CHECK(exsum_host_sum(w, 3, 0, 1, &out, nullptr) == EXSUM_OK && out == 1.0);
  std::printf("host ok (%s)\n", exsum_version());
  return 0;
}

static int device_checks() {
  // exact_sum of a host array through the device (the call a reference user makes)
  const size_t n = 10'000'003;
  std::vector<double> x(n);
  CHECK(exsum_host_gen(3, 7, n, 0, n, x.data()) == EXSUM_OK);
  exsum_context *ctx = exsum_context_create(0, size_t{64} << 20);
  CHECK(ctx != nullptr);
  double dev = 0, host = 0;
  exsum_partial rec;
  CHECK(exsum_context_sum(ctx, x.data(), n, &dev, &rec) == EXSUM_OK);
  exsum_large *L = exsum_large_new();
  CHECK(exsum_large_add_array(L, x.data(), n) == EXSUM_OK);
  CHECK(exsum_large_round(L, &host) == EXSUM_OK);
  exsum_large_free(L);
  CHECK(bits(dev) == bits(host));
  // the same call split between the device and 3 host workers, and device only
  uint64_t dterms = 0, hterms = 0;
  CHECK(exsum_context_set_host_threads(ctx, 3) == EXSUM_OK);
  CHECK(exsum_context_sum(ctx, x.data(), n, &dev, nullptr) == EXSUM_OK && bits(dev) == bits(host));
  CHECK(exsum_context_last_split(ctx, &dterms, &hterms) == EXSUM_OK && dterms + hterms == n);
  CHECK(exsum_context_set_host_threads(ctx, 0) == EXSUM_OK);
  CHECK(exsum_context_sum(ctx, x.data(), n, &dev, nullptr) == EXSUM_OK && bits(dev) == bits(host));
  CHECK(exsum_context_last_split(ctx, &dterms, &hterms) == EXSUM_OK && dterms == n);
  // segmented host arrays: three segments, one empty
  const uint64_t offs[4] = {0, 1000, 1000, n};
  double sums[3];
  CHECK(exsum_context_sum_segmented(ctx, x.data(), offs, 3, sums, nullptr) == EXSUM_OK);
  double s0 = 0;
  CHECK(exsum_host_sum(x.data(), 1000, 0, 1, &s0, nullptr) == EXSUM_OK && bits(sums[0]) == bits(s0));
  CHECK(bits(sums[1]) == 0);
  exsum_context_free(ctx);
  std::printf("device ok: %016llx\n", static_cast<unsigned long long>(bits(dev)));
  return 0;
}

int main(int argc, char **argv) {
  if (host_checks()) return 1;
  if (argc > 1 && std::strcmp(argv[1], "--device") == 0 && device_checks()) return 1;
  return 0;
}
