// Config 1 in a C loop: exact_sum(x, 1000, small) of the compiled reference (oracle/_ref,
// ref_exact_sum) vs exsum_exact_sum, same 1000 U[-1,1) terms, plus a 20,000-case random
// exactness sweep of the two.  Probe, not product:
//   g++ -O2 scripts/probes/small_exact_sum.cpp -o /tmp/s -ldl && /tmp/s oracle/_ref/libexsum_ref.so paper_1505_05571_b200/lib/libexsum_b200.so
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <random>
#include <dlfcn.h>
typedef double (*rfn_t)(const double*, size_t, int);
typedef int (*fn_t)(const double*, size_t, int, double*);
int main(int argc, char** argv) {
  void* hr = dlopen(argv[1], RTLD_NOW); void* ho = dlopen(argv[2], RTLD_NOW);
  rfn_t r = (rfn_t)dlsym(hr, "ref_exact_sum"); fn_t f = (fn_t)dlsym(ho, "exsum_exact_sum");
  std::mt19937_64 g(1); std::uniform_real_distribution<double> U(-1, 1);
  double x[1000]; for (auto& v : x) v = U(g);
  int reps = 200000; double out = 0, ro = 0;
  for (int i = 0; i < 1000; ++i) ro = r(x, 1000, 0);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) ro = r(x, 1000, 0);
  auto t1 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) f(x, 1000, 0, &out);
  auto t2 = std::chrono::steady_clock::now();
  uint64_t a, b; memcpy(&a, &ro, 8); memcpy(&b, &out, 8);
  printf("reference %.3f us, ours %.3f us, bits %s\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / reps, std::chrono::duration<double, std::micro>(t2 - t1).count() / reps, a == b ? "equal" : "DIFFER");
  // exactness sweep: random lengths and distributions
  int bad = 0;
  for (int t = 0; t < 20000; ++t) {
    size_t n = g() % 5000;
    static double y[5000];
    int kind = t % 5;
    for (size_t i = 0; i < n; ++i) {
      uint64_t u = g();
      if (kind == 0) y[i] = U(g);
      else if (kind == 1) { memcpy(&y[i], &u, 8); if (((u >> 52) & 0x7FF) == 0x7FF) y[i] = 1.0; }
      else if (kind == 2) y[i] = (g() & 1 ? -1 : 1) * std::ldexp(1.0 + U(g), (int)(g() % 200) - 100);
      else if (kind == 3) { u &= 0x800FFFFFFFFFFFFFull; memcpy(&y[i], &u, 8); }
      else { memcpy(&y[i], &u, 8); }
    }
    double o1 = r(y, n, 0), o2; f(y, n, 0, &o2);
    uint64_t c1, c2; memcpy(&c1, &o1, 8); memcpy(&c2, &o2, 8);
    if (c1 != c2) { if (bad < 5) printf("mismatch t=%d kind=%d n=%zu %016llx %016llx\n", t, kind, n, (unsigned long long)c1, (unsigned long long)c2); ++bad; }
  }
  printf("sweep mismatches: %d\n", bad);
}
