// small_bench.cpp — config 1 (SmallAccumulator, N = 1000) in C: this library's
// exsum_small_* against the compiled reference (oracle/_ref shim), no Python
// call overhead.  Probe, not product.
//   g++ -O2 -std=c++17 -I../../include small_bench.cpp -o small_bench -ldl
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <chrono>

#include "exsum_b200.h"

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int main(int argc, char **argv) {
  const char *ours_so = argc > 1 ? argv[1] : "../../paper_1505_05571_b200/lib/libexsum_b200.so";
  const char *ref_so = argc > 2 ? argv[2] : "../../oracle/_ref/libexsum_ref.so";
  void *ho = dlopen(ours_so, RTLD_NOW), *hr = dlopen(ref_so, RTLD_NOW);
  if (!ho || !hr) {
    printf("dlopen failed: %s\n", dlerror());
    return 1;
  }
  auto o_init = (int (*)(exsum_small *))dlsym(ho, "exsum_small_init");
  auto o_add = (int (*)(exsum_small *, const double *, size_t))dlsym(ho, "exsum_small_add_array");
  auto o_round = (int (*)(exsum_small *, double *))dlsym(ho, "exsum_small_round");
  auto r_init = (void (*)(void *))dlsym(hr, "ref_small_init");
  auto r_add = (void (*)(void *, const double *, size_t))dlsym(hr, "ref_small_add_array");
  auto r_round = (double (*)(void *))dlsym(hr, "ref_small_round");
  double x[1000];
  for (int i = 0; i < 1000; ++i) x[i] = (mix(i + 1) >> 11) * 0x1.0p-53 * 2.0 - 1.0;
  exsum_small a;
  alignas(16) unsigned char r[560];
  double so = 0, sr = 0;
  const int reps = 200000;
  for (int t = 0; t < 3; ++t) {
    double t0 = now();
    for (int k = 0; k < reps; ++k) {
      o_init(&a);
      o_add(&a, x, 1000);
      double v;
      o_round(&a, &v);
      so += v;
    }
    double t1 = now();
    for (int k = 0; k < reps; ++k) {
      r_init(r);
      r_add(r, x, 1000);
      sr += r_round(r);
    }
    double t2 = now();
    printf("ours %.3f us/sum   reference %.3f us/sum   (%s)\n", (t1 - t0) / reps * 1e6,
           (t2 - t1) / reps * 1e6, so == sr ? "same bits" : "DIFFERENT");
  }
}
