// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg load the resulting libexsum_ref.so, and only as a checker or
// as the timed CPU baseline.  None of the reference sources are copied here;
// this file only forwards plain pointers to the reference's C++ API:
//
//   exsum::SmallAccumulator  small_accumulator.hpp:47-103
//   exsum::LargeAccumulator  large_accumulator.hpp:43-104
//   exsum::exact_sum / parallel_exact_sum / exact_mean / sqnorm / dot
//                            vector_ops.hpp:35-75
//   exsum::sum_ordered / sum_unordered / sum_kahan   baselines.hpp:21-35
//   exsum::generate          generator.hpp:25-60
//   exsum::read_values / write_values   io.hpp:31-37
//
// The SmallAccumulator is standard-layout and trivially copyable (560 B),
// so it crosses this boundary as raw bytes.

#include <cstdint>
#include <cstring>
#include <new>
#include <span>
#include <stdexcept>
#include <type_traits>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include <cstdlib>
#include <string>

#include "exsum/baselines.hpp"
#include "exsum/io.hpp"
#include "exsum/generator.hpp"
#include "exsum/large_accumulator.hpp"
#include "exsum/small_accumulator.hpp"
#include "exsum/vector_ops.hpp"

using exsum::LargeAccumulator;
using exsum::SmallAccumulator;

static_assert(std::is_trivially_copyable_v<SmallAccumulator>);
static_assert(sizeof(SmallAccumulator) == 560);

namespace {

SmallAccumulator load_small(const void *p) {
  SmallAccumulator a;
  std::memcpy(static_cast<void *>(&a), p, sizeof a);
  return a;
}

void store_small(void *p, const SmallAccumulator &a) {
  std::memcpy(p, static_cast<const void *>(&a), sizeof a);
}

std::span<const double> span_of(const double *x, std::size_t n) {
  return {x, n};
}

}  // namespace

extern "C" {

int ref_small_sizeof(void) { return static_cast<int>(sizeof(SmallAccumulator)); }

void ref_small_init(void *acc) { store_small(acc, SmallAccumulator{}); }

void ref_small_add(void *acc, double v) {
  SmallAccumulator a = load_small(acc);
  a.add(v);
  store_small(acc, a);
}

void ref_small_add_array(void *acc, const double *x, std::size_t n) {
  SmallAccumulator a = load_small(acc);
  a.add(span_of(x, n));
  store_small(acc, a);
}

void ref_small_add_inf_nan(void *acc, std::uint64_t bits) {
  SmallAccumulator a = load_small(acc);
  a.add_inf_nan(bits);
  store_small(acc, a);
}

int ref_small_carry_propagate(void *acc) {
  SmallAccumulator a = load_small(acc);
  const int top = a.carry_propagate();
  store_small(acc, a);
  return top;
}

void ref_small_merge(void *dst, const void *src) {
  SmallAccumulator a = load_small(dst);
  a.merge(load_small(src));
  store_small(dst, a);
}

double ref_small_round(void *acc) {
  SmallAccumulator a = load_small(acc);
  const double r = a.round();
  store_small(acc, a);
  return r;
}

// Returns 0 on success, 1 when the reference throws std::invalid_argument.
int ref_small_mean(void *acc, std::uint64_t n, double *out) {
  SmallAccumulator a = load_small(acc);
  try {
    *out = a.mean(n);
  } catch (const std::invalid_argument &) {
    return 1;
  }
  store_small(acc, a);
  return 0;
}

void *ref_large_new(void) { return new (std::nothrow) LargeAccumulator(); }
void ref_large_free(void *p) { delete static_cast<LargeAccumulator *>(p); }
void ref_large_add(void *p, double v) { static_cast<LargeAccumulator *>(p)->add(v); }
void ref_large_add_array(void *p, const double *x, std::size_t n) {
  static_cast<LargeAccumulator *>(p)->add(span_of(x, n));
}
void ref_large_drain(void *p) { static_cast<LargeAccumulator *>(p)->drain(); }
double ref_large_round(void *p) { return static_cast<LargeAccumulator *>(p)->round(); }
void ref_large_small(void *p, void *out_small) {
  store_small(out_small, static_cast<LargeAccumulator *>(p)->small());
}
int ref_large_count(void *p, int ix) {
  return static_cast<LargeAccumulator *>(p)->counts()[static_cast<std::size_t>(ix)];
}
int ref_large_chunk_in_use(void *p, int ix) {
  return static_cast<LargeAccumulator *>(p)->chunk_in_use(ix) ? 1 : 0;
}
std::uint64_t ref_large_chunk_word(void *p, int ix) {
  return static_cast<LargeAccumulator *>(p)->chunk_word(ix);
}
int ref_large_chunks_in_use(void *p) {
  return static_cast<LargeAccumulator *>(p)->chunks_in_use();
}

// method: 0 = small, 1 = large (exsum::ExactMethod order).
double ref_exact_sum(const double *x, std::size_t n, int method) {
  return exsum::exact_sum(span_of(x, n), method == 0 ? exsum::ExactMethod::small
                                                      : exsum::ExactMethod::large);
}

int ref_exact_mean(const double *x, std::size_t n, int method, double *out) {
  try {
    *out = exsum::exact_mean(span_of(x, n), method == 0 ? exsum::ExactMethod::small
                                                         : exsum::ExactMethod::large);
  } catch (const std::invalid_argument &) {
    return 1;
  }
  return 0;
}

double ref_parallel_exact_sum(const double *x, std::size_t n, int parts,
                              std::size_t large_threshold) {
  exsum::ParallelPlan plan;
  plan.parts = parts;
  plan.large_threshold = large_threshold;
  return exsum::parallel_exact_sum(span_of(x, n), plan);
}

double ref_parallel_exact_sum_serial(const double *x, std::size_t n, int parts,
                                     std::size_t large_threshold) {
  exsum::ParallelPlan plan;
  plan.parts = parts;
  plan.large_threshold = large_threshold;
  return exsum::parallel_exact_sum_serial(span_of(x, n), plan);
}

// Canonical 67-chunk state of the exact sum: large accumulator over the
// values, drain, carry_propagate (history-independent form).
// Also returns the embedded small accumulator's inf/nan bits.
int ref_canonical(const double *x, std::size_t n, std::int64_t *chunks67,
                  std::uint64_t *inf_bits, std::uint64_t *nan_bits) {
  LargeAccumulator *acc = new LargeAccumulator();
  acc->add(span_of(x, n));
  acc->drain();
  SmallAccumulator s = acc->small();
  delete acc;
  const int top = s.carry_propagate();
  for (int i = 0; i < exsum::kSmallChunks; ++i) chunks67[i] = s.chunks()[static_cast<std::size_t>(i)];
  *inf_bits = s.inf_bits();
  *nan_bits = s.nan_bits();
  return top;
}

// One exact_sum(large) per segment, OpenMP over segments (BASELINE.md §2,
// config 5).  offsets has nseg + 1 entries.
void ref_segmented_sum(const double *x, const std::uint64_t *offsets,
                       std::size_t nseg, double *out, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  const long long ns = static_cast<long long>(nseg);
#pragma omp parallel for schedule(dynamic, 16)
  for (long long i = 0; i < ns; ++i) {
    const std::uint64_t b = offsets[i], e = offsets[i + 1];
    out[i] = exsum::exact_sum(span_of(x + b, e - b), exsum::ExactMethod::large);
  }
}

void ref_set_threads(int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
}

int ref_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// read_values / write_values: 0 on success, 1 when the reference throws; the
// message is copied to msg (msg_len bytes).  *out is malloc'ed (free with
// ref_free).
int ref_read_values(const char *path, int format, double **out, std::size_t *n, char *msg,
                    std::size_t msg_len) {
  try {
    const std::vector<double> v =
        exsum::read_values(path, format ? exsum::FileFormat::text : exsum::FileFormat::bin);
    *n = v.size();
    *out = static_cast<double *>(std::malloc(v.empty() ? 8 : v.size() * 8));
    if (!v.empty()) std::memcpy(*out, v.data(), v.size() * 8);
    return 0;
  } catch (const std::exception &e) {
    std::snprintf(msg, msg_len, "%s", e.what());
    return 1;
  }
}

int ref_write_values(const char *path, const double *x, std::size_t n, int format) {
  try {
    exsum::write_values(path, span_of(x, n),
                        format ? exsum::FileFormat::text : exsum::FileFormat::bin);
    return 0;
  } catch (const std::exception &) {
    return 1;
  }
}

void ref_free(void *p) { std::free(p); }

double ref_sqnorm(const double *x, std::size_t n, int method) {
  return exsum::sqnorm(span_of(x, n), static_cast<exsum::SumMethod>(method));
}

int ref_dot(const double *a, const double *b, std::size_t na, std::size_t nb,
            int method, double *out) {
  try {
    *out = exsum::dot(span_of(a, na), span_of(b, nb), static_cast<exsum::SumMethod>(method));
  } catch (const std::invalid_argument &) {
    return 1;
  }
  return 0;
}

double ref_sum_ordered(const double *x, std::size_t n) { return exsum::sum_ordered(span_of(x, n)); }
double ref_sum_unordered(const double *x, std::size_t n) { return exsum::sum_unordered(span_of(x, n)); }
double ref_sum_kahan(const double *x, std::size_t n) { return exsum::sum_kahan(span_of(x, n)); }

// The reference's benchmark-data generator (generator.cpp:23-45).
int ref_generate(std::uint64_t n, std::uint64_t seed, int permute, double *out) {
  exsum::GeneratorSpec spec;
  spec.n = n;
  spec.seed = seed;
  spec.permute = permute != 0;
  try {
    const std::vector<double> v = exsum::generate(spec);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  } catch (const std::invalid_argument &) {
    return 1;
  }
  return 0;
}

}  // extern "C"
