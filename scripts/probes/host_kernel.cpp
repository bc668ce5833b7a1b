// host_kernel.cpp — single-thread rate of the host superaccumulator kernel
// (csrc/host_sum.cpp) against a plain streaming read, on in-cache and
// out-of-cache arrays.  Probe, not product.
//   g++ -O3 -std=c++17 -I../../include -I../../paper_1505_05571_b200/csrc \
//       host_kernel.cpp ../../paper_1505_05571_b200/csrc/host_sum.cpp \
//       ../../paper_1505_05571_b200/csrc/host_accumulators.cpp -o host_kernel -pthread
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "host_sum.h"

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// T threads, each summing its contiguous slice of x[0..n) once per rep: aggregate GB/s.
static double threaded(const std::vector<uint64_t> &x, size_t n, int T, int reps) {
  std::vector<exsum_host::Acc *> acc(T);
  for (auto &a : acc) a = new exsum_host::Acc;
  double best = 1e9;
  for (int r = 0; r < reps; ++r) {
    double t0 = now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        size_t b = n * t / T, e = n * (t + 1) / T;
        acc[t]->reset();
        acc[t]->add(reinterpret_cast<const double *>(x.data()) + b, e - b, b);
      });
    for (auto &h : th) h.join();
    double el = now() - t0;
    if (el < best) best = el;
  }
  for (auto *a : acc) delete a;
  return 8.0 * n / best / 1e9;
}

int main(int argc, char **argv) {
  size_t big = argc > 1 ? strtoull(argv[1], 0, 10) : 50000000;
  if (argc > 2) {  // threaded mode: host_kernel N T
    int T = atoi(argv[2]);
    std::vector<uint64_t> x(big);
    for (int cfg : {2, 3, 4}) {
      for (size_t i = 0; i < big; ++i) {
        uint64_t h = mix(i * 0x9E3779B97F4A7C15ull + cfg), b;
        if (cfg == 2) { double d = (h >> 11) * 0x1.0p-53; memcpy(&b, &d, 8); }
        else if (cfg == 3) { uint64_t e = 1 + (mix(h) % 2046); if (mix(h + 1) % 100 == 0) e = 0; b = (h & 0x800FFFFFFFFFFFFFull) | (e << 52); }
        else { uint64_t e = 1023 - 66 + (h % 133); b = (h & 0x800FFFFFFFFFFFFFull) | (e << 52); }
        x[i] = b;
      }
      printf("cfg%d T=%d: %.2f GB/s\n", cfg, T, threaded(x, big, T, 3));
      fflush(stdout);
    }
    return 0;
  }
  std::vector<uint64_t> x(big);
  auto *acc = new exsum_host::Acc;
  for (int cfg : {2, 3, 4, 6}) {
    for (size_t i = 0; i < big; ++i) {
      uint64_t h = mix(i * 0x9E3779B97F4A7C15ull + cfg);
      double d;
      if (cfg == 2) d = (h >> 11) * 0x1.0p-53;
      else if (cfg == 3 || cfg == 6) { uint64_t e = 1 + (mix(h) % 2046); if (cfg == 3 && mix(h+1) % 100 == 0) e = 0; uint64_t b = (h & 0x800FFFFFFFFFFFFFull) | (e << 52); memcpy(&d, &b, 8); }
      else { uint64_t e = 1023 - 66 + (h % 133); uint64_t b = (h & 0x800FFFFFFFFFFFFFull) | (e << 52); memcpy(&d, &b, 8); }
      memcpy(&x[i], &d, 8);
    }
    for (size_t n : {size_t(40000), big}) {
      size_t reps = n < big ? 2000 : 3;
      double best = 1e9, bestr = 1e9;
      uint64_t sink = 0;
      for (int t = 0; t < 3; ++t) {
        acc->reset();
        double t0 = now();
        for (size_t r = 0; r < reps; ++r) acc->add(reinterpret_cast<double *>(x.data()), n, 0);
        double el = now() - t0;
        if (el < best) best = el;
        t0 = now();
        for (size_t r = 0; r < reps; ++r) {
          uint64_t s = 0;
          for (size_t i = 0; i < n; ++i) s += x[i];
          sink += s;
        }
        el = now() - t0;
        if (el < bestr) bestr = el;
      }
      exsum_partial p;
      acc->finish(&p);
      printf("cfg%d n=%zu: kernel %.2f GB/s (%.2f ns/term)  plain read %.2f GB/s %llu\n", cfg, n,
             8.0 * n * reps / best / 1e9, best / (n * reps) * 1e9, 8.0 * n * reps / bestr / 1e9,
             (unsigned long long)(sink & 1));
    }
  }
}
