// A reference caller, unchanged except for the namespace alias: the SPEC.md
// per-operation examples and acceptance checks written against the reference's
// C++ API (SmallAccumulator, LargeAccumulator, exact_sum, exact_mean, sqnorm,
// dot, parallel_exact_sum, read/write_values, generate), compiled against
// include/exsum_b200.hpp.  --device adds DeviceContext (the B200 path).
//
//   g++ -std=c++20 -Iinclude tests/cpp/dropin.cpp -Lpaper_1505_05571_b200/lib -lexsum_b200
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <limits>
#include <random>
#include <stdexcept>
#include <vector>

#include "exsum_b200.hpp"

namespace exsum = exsum_b200;  // the only change a reference caller makes

static std::uint64_t bits(double v) {
  std::uint64_t b;
  std::memcpy(&b, &v, 8);
  return b;
}
static double from_bits(std::uint64_t b) {
  double v;
  std::memcpy(&v, &b, 8);
  return v;
}

#define CHECK(cond)                                                          \
  do {                                                                       \
    if (!(cond)) {                                                           \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      return 1;                                                              \
    }                                                                        \
  } while (0)

template <class F>
static bool throws_invalid(F f) {
  try {
    f();
  } catch (const std::invalid_argument &) {
    return true;
  }
  return false;
}

static int host() {
  // SmallAccumulator
  {
    exsum::SmallAccumulator a;
    a.add(1.0);
    CHECK(a.chunks()[32] == (std::int64_t{1} << 51));
    exsum::SmallAccumulator b;
    b.add(from_bits(1));  // 2^-1074
    CHECK(b.chunks()[0] == 2);
    exsum::SmallAccumulator c;
    c.add(-0.0);
    for (auto v : c.chunks()) CHECK(v == 0);
    std::vector<double> ones(5000, 1.0);
    exsum::SmallAccumulator d;
    d.add(ones);
    CHECK(d.round() == 5000.0);
    const double cancel[3] = {1e15, -1e15, 0.1};
    exsum::SmallAccumulator e;
    e.add(cancel);
    CHECK(e.round() == 0.1);
    exsum::SmallAccumulator f;
    f.add(INFINITY);
    f.add(-INFINITY);
    CHECK(bits(f.round()) == 0x7FF8000000000000ull);
    CHECK(throws_invalid([&] { d.mean(0); }));
    exsum::SmallAccumulator g;
    g.add(1e16);
    exsum::SmallAccumulator h;
    h.add(1.0);
    h.add(-1e16);
    g.merge(h);
    CHECK(g.round() == 1.0);
  }
  // LargeAccumulator
  {
    exsum::LargeAccumulator L;
    L.add(1.0);
    CHECK(L.count(0x3FF) == 4095 && L.chunk_in_use(0x3FF) && L.chunks_in_use() == 1);
    std::vector<double> ones(4097, 1.0);
    exsum::LargeAccumulator M;
    M.add(ones);
    CHECK(M.round() == 4097.0);
    const double w[3] = {1e16, 1.0, -1e16};
    exsum::LargeAccumulator N;
    N.add(w);
    CHECK(N.round() == 1.0);
  }
  // vector_ops: exact_sum / sum / sqnorm / dot / exact_mean / parallel_exact_sum
  {
    const double ob[4] = {1.5e308, 1.5e308, -1.5e308, -0.5e308};  // overflow bypass
    CHECK(bits(exsum::exact_sum(ob, exsum::ExactMethod::large)) == 0x7fe1ccf385ebc8a0ull);
    CHECK(bits(exsum::exact_sum(ob, exsum::ExactMethod::small)) == 0x7fe1ccf385ebc8a0ull);
    CHECK(exsum::parse_method("large") == exsum::SumMethod::large);
    CHECK(throws_invalid([] { exsum::parse_method("bogus"); }));
    CHECK(throws_invalid([] { exsum::exact_mean({}, exsum::ExactMethod::large); }));
    const double a3[3] = {3.0, 4.0, 0.0}, b2[2] = {1.0, 2.0};
    CHECK(exsum::sqnorm(a3, exsum::SumMethod::large) == 25.0);
    CHECK(throws_invalid([&] { exsum::dot(a3, b2, exsum::SumMethod::large); }));
    CHECK(throws_invalid([&] { exsum::sum(a3, exsum::SumMethod::kahan); }));
    std::mt19937_64 rng(7);
    std::vector<double> x(200'003);
    for (auto &v : x) {
      std::uint64_t r = rng();
      r = (r & 0x800FFFFFFFFFFFFFull) | (std::uint64_t(1 + rng() % 2046) << 52);
      v = from_bits(r);
    }
    const double want = exsum::exact_sum(x, exsum::ExactMethod::small);
    CHECK(bits(exsum::exact_sum(x, exsum::ExactMethod::large)) == bits(want));
    CHECK(bits(exsum::sum(x, exsum::SumMethod::large)) == bits(want));
    for (int parts : {1, 2, 3, 8, 16})
      CHECK(bits(exsum::parallel_exact_sum(x, {parts})) == bits(want));
    CHECK(bits(exsum::parallel_exact_sum_serial(x)) == bits(want));
    std::vector<double> y(1000, 3.0);
    CHECK(exsum::exact_mean(y, exsum::ExactMethod::large) == 3.0);
    CHECK(exsum::exact_mean(y, exsum::ExactMethod::small) == 3.0);
    // generator: zero exact sum
    const auto g = exsum::generate({1'000'000, 3, true});
    CHECK(bits(exsum::exact_sum(g, exsum::ExactMethod::large)) == 0);
    CHECK(throws_invalid([] { exsum::generate({7, 1, false}); }));
    // io round trip
    const auto dir = std::filesystem::temp_directory_path();
    for (auto fmt : {exsum::FileFormat::bin, exsum::FileFormat::text}) {
      const auto p = dir / (fmt == exsum::FileFormat::bin ? "dropin.bin" : "dropin.txt");
      exsum::write_values(p, x, fmt);
      const auto back = exsum::read_values(p, fmt);
      CHECK(back.size() == x.size() && std::memcmp(back.data(), x.data(), 8 * x.size()) == 0);
      std::filesystem::remove(p);
    }
    bool io_error = false;
    try {
      exsum::read_values(dir / "no-such-file.bin", exsum::FileFormat::bin);
    } catch (const std::runtime_error &) {
      io_error = true;
    }
    CHECK(io_error);
  }
  std::printf("dropin host ok\n");
  return 0;
}

static int device() {
  exsum::DeviceContext ctx(0);
  const auto g = exsum::generate({8'000'000, 5, true});
  CHECK(bits(ctx.exact_sum(g)) == 0);
  std::mt19937_64 rng(9);
  std::vector<double> x(6'000'001);
  for (auto &v : x) v = std::ldexp(double(rng() >> 11), int(rng() % 200) - 150) * (rng() & 1 ? 1 : -1);
  const double want = exsum::exact_sum(x, exsum::ExactMethod::large);
  CHECK(bits(ctx.exact_sum(x)) == bits(want));
  const auto [dev, host] = ctx.last_split();
  CHECK(dev + host == x.size() && dev > 0);
  ctx.set_host_threads(0);
  CHECK(bits(ctx.exact_sum(x)) == bits(want));
  CHECK(bits(ctx.exact_mean(x)) == bits(exsum::exact_mean(x, exsum::ExactMethod::large)));
  const std::vector<std::uint64_t> offs = {0, 1000, 1000, 3'000'000, x.size()};
  const auto segs = ctx.exact_sum_segmented(x, offs);
  CHECK(segs.size() == 4 && bits(segs[1]) == 0);
  CHECK(bits(segs[2]) == bits(exsum::exact_sum(std::span<const double>(x).subspan(1000, 2'999'000),
                                               exsum::ExactMethod::large)));
  std::printf("dropin device ok\n");
  return 0;
}

int main(int argc, char **argv) {
  if (host()) return 1;
  if (argc > 1 && std::strcmp(argv[1], "--device") == 0 && device()) return 1;
  return 0;
}
