// exsum_b200.hpp — C++20 mirror of the reference's summation API over the C ABI.
//
// The reference (exsum, /root/reference/proj/include/exsum) is a C++ library;
// its callers use SmallAccumulator, LargeAccumulator, exact_sum, exact_mean,
// sqnorm, dot, parallel_exact_sum, read_values/write_values and generate.  This
// header-only layer gives them the same names, argument meanings and error
// behaviour (std::invalid_argument / std::runtime_error) in namespace
// exsum_b200, implemented on include/exsum_b200.h (libexsum_b200.so), so a
// caller switches libraries with a namespace alias:
//
//     namespace exsum = exsum_b200;   // was: #include "exsum/vector_ops.hpp"
//
// plus DeviceContext for the B200 path of host-resident arrays (exact_sum of a
// std::span through the device and the host cores) — the drop-in for
// exact_sum on large arrays.  Results are bit-identical to the reference.
#ifndef EXSUM_B200_HPP_
#define EXSUM_B200_HPP_

#include <cstddef>
#include <cstdint>
#include <filesystem>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "exsum_b200.h"

namespace exsum_b200 {

inline constexpr int kSmallChunks = EXSUM_SMALL_CHUNKS;      // small_accumulator.hpp:32
inline constexpr int kSmallCarryTerms = EXSUM_SMALL_CARRY_TERMS;
inline constexpr int kLargeChunks = EXSUM_LARGE_CHUNKS;      // large_accumulator.hpp:27
inline constexpr std::size_t kLargeMethodThreshold = 1000;  // vector_ops.hpp:30

namespace detail {
inline void check(int status, const char *what) {
  switch (status) {
    case EXSUM_OK:
      return;
    case EXSUM_EINVAL:
      throw std::invalid_argument(what);
    case EXSUM_EIO:
      throw std::runtime_error(exsum_io_error());
    default:
      throw std::runtime_error(std::string(what) + ": exsum_b200 status " +
                               std::to_string(status));
  }
}
}  // namespace detail

// exsum::SmallAccumulator (small_accumulator.hpp:45-104): the same 560 bytes.
class SmallAccumulator {
 public:
  SmallAccumulator() { exsum_small_init(&s_); }
  void add(double v) { exsum_small_add(&s_, v); }
  void add(std::span<const double> values) {
    exsum_small_add_array(&s_, values.data(), values.size());
  }
  void merge(const SmallAccumulator &other) { exsum_small_merge(&s_, &other.s_); }
  double round() {
    double out;
    exsum_small_round(&s_, &out);
    return out;
  }
  // throws std::invalid_argument for n == 0 (small_accumulator.cpp:351-353)
  double mean(std::uint64_t n) {
    double out;
    detail::check(exsum_small_mean(&s_, n, &out), "mean: n must be positive");
    return out;
  }
  void add_inf_nan(std::uint64_t bits) { exsum_small_add_inf_nan(&s_, bits); }
  int carry_propagate() { return exsum_small_carry_propagate(&s_); }
  std::span<const std::int64_t, kSmallChunks> chunks() const {
    return std::span<const std::int64_t, kSmallChunks>(s_.chunk, kSmallChunks);
  }
  int adds_until_propagate() const { return s_.adds_until_propagate; }
  std::uint64_t inf_bits() const { return s_.inf_bits; }
  std::uint64_t nan_bits() const { return s_.nan_bits; }

  const exsum_small &raw() const { return s_; }
  static SmallAccumulator from_raw(const exsum_small &s) {
    SmallAccumulator a;
    a.s_ = s;
    return a;
  }

 private:
  exsum_small s_;
};
static_assert(sizeof(SmallAccumulator) == 560, "layout of exsum::SmallAccumulator");

// exsum::LargeAccumulator (large_accumulator.hpp:40-104).
class LargeAccumulator {
 public:
  LargeAccumulator() : p_(exsum_large_new()) {
    if (!p_) throw std::bad_alloc();
  }
  ~LargeAccumulator() { exsum_large_free(p_); }
  LargeAccumulator(const LargeAccumulator &) = delete;
  LargeAccumulator &operator=(const LargeAccumulator &) = delete;
  LargeAccumulator(LargeAccumulator &&o) noexcept : p_(std::exchange(o.p_, nullptr)) {}

  void add(double v) { exsum_large_add(p_, v); }
  void add(std::span<const double> values) {
    exsum_large_add_array(p_, values.data(), values.size());
  }
  void drain() { exsum_large_drain(p_); }
  double round() {
    double out;
    exsum_large_round(p_, &out);
    return out;
  }
  double mean(std::uint64_t n) {
    double out;
    detail::check(exsum_large_mean(p_, n, &out), "mean: n must be positive");
    return out;
  }
  // a copy of the embedded small accumulator (the reference returns a reference)
  SmallAccumulator small() const {
    exsum_small s;
    exsum_large_small(p_, &s);
    return SmallAccumulator::from_raw(s);
  }
  // counts()[ix] of the reference: adds left before the chunk transfers, -1 unused
  int count(int ix) const {
    int c = -1;
    detail::check(exsum_large_count(p_, ix, &c), "count: index out of range");
    return c;
  }
  bool chunk_in_use(int ix) const { return exsum_large_chunk_in_use(p_, ix) != 0; }
  std::uint64_t chunk_word(int ix) const {
    std::uint64_t w = 0;
    detail::check(exsum_large_chunk_word(p_, ix, &w), "chunk_word: index out of range");
    return w;
  }
  int chunks_in_use() const { return exsum_large_chunks_in_use(p_); }

 private:
  exsum_large *p_;
};

// vector_ops.hpp:23-75.  The inexact baselines (ordered / unordered / kahan,
// baselines.cpp) are out of scope: sum/sqnorm/dot with those methods throw.
enum class SumMethod { small, large, ordered, unordered, kahan };
enum class ExactMethod { small, large };

inline SumMethod parse_method(std::string_view name) {
  if (name == "small") return SumMethod::small;
  if (name == "large") return SumMethod::large;
  if (name == "ordered") return SumMethod::ordered;
  if (name == "unordered") return SumMethod::unordered;
  if (name == "kahan") return SumMethod::kahan;
  throw std::invalid_argument("unknown method: " + std::string(name));
}

inline std::string_view method_name(SumMethod m) {
  switch (m) {
    case SumMethod::small: return "small";
    case SumMethod::large: return "large";
    case SumMethod::ordered: return "ordered";
    case SumMethod::unordered: return "unordered";
    case SumMethod::kahan: return "kahan";
  }
  return "?";
}

inline double exact_sum(std::span<const double> values, ExactMethod method) {
  double out;
  detail::check(exsum_exact_sum(values.data(), values.size(),
                                method == ExactMethod::small ? 0 : 1, &out),
                "exact_sum");
  return out;
}

namespace detail {
inline ExactMethod exact_only(SumMethod m) {
  if (m == SumMethod::small) return ExactMethod::small;
  if (m == SumMethod::large) return ExactMethod::large;
  throw std::invalid_argument("method " + std::string(method_name(m)) +
                              ": only the exact methods are provided (baselines are out of scope)");
}
}  // namespace detail

inline double sum(std::span<const double> values, SumMethod method) {
  return exact_sum(values, detail::exact_only(method));
}

// the exact sum of the rounded squares / products (vector_ops.cpp:143-155);
// dot throws std::invalid_argument on a length mismatch (:150-152)
inline double sqnorm(std::span<const double> values, SumMethod method) {
  detail::exact_only(method);
  double out;
  detail::check(exsum_sqnorm(values.data(), values.size(), &out), "sqnorm");
  return out;
}

inline double dot(std::span<const double> a, std::span<const double> b, SumMethod method) {
  detail::exact_only(method);
  double out;
  detail::check(exsum_dot(a.data(), a.size(), b.data(), b.size(), &out),
                "dot: vectors must have equal length");
  return out;
}

// exact_mean (vector_ops.cpp:157-170): throws std::invalid_argument when empty
inline double exact_mean(std::span<const double> values, ExactMethod method) {
  if (values.empty()) throw std::invalid_argument("exact_mean: empty input");
  if (method == ExactMethod::small) {
    SmallAccumulator acc;
    acc.add(values);
    return acc.mean(values.size());
  }
  exsum_partial rec;
  detail::check(exsum_host_sum(values.data(), values.size(), 0, 1, nullptr, &rec), "exact_mean");
  double out;
  detail::check(exsum_small_mean(&rec.acc, values.size(), &out), "exact_mean");
  return out;
}

// ParallelPlan / parallel_exact_sum (vector_ops.hpp:55-75): `parts` host
// threads with this library's host kernel (exsum_host_sum); same bits for any
// parts, like the reference's split-merge.
struct ParallelPlan {
  int parts = 1;
  std::size_t large_threshold = kLargeMethodThreshold;  // accepted for parity
};

inline double parallel_exact_sum(std::span<const double> values, const ParallelPlan &plan = {}) {
  double out;
  detail::check(exsum_host_sum(values.data(), values.size(), 0, plan.parts < 1 ? 1 : plan.parts,
                               &out, nullptr),
                "parallel_exact_sum");
  return out;
}

inline double parallel_exact_sum_serial(std::span<const double> values,
                                        const ParallelPlan & = {}) {
  return exact_sum(values, ExactMethod::large);
}

// io.hpp: FileFormat, parse_format, read_values, write_values (io.cpp:71-159).
enum class FileFormat { bin, text };

inline FileFormat parse_format(std::string_view name) {
  const int f = exsum_parse_format(std::string(name).c_str());
  if (f < 0) throw std::invalid_argument("unknown format: " + std::string(name));
  return f == EXSUM_FORMAT_BIN ? FileFormat::bin : FileFormat::text;
}

inline std::vector<double> read_values(const std::filesystem::path &path, FileFormat format) {
  double *v = nullptr;
  std::size_t n = 0;
  detail::check(exsum_read_values(path.c_str(), format == FileFormat::bin ? EXSUM_FORMAT_BIN
                                                                          : EXSUM_FORMAT_TEXT,
                                  &v, &n),
                "read_values");
  std::vector<double> out(v, v + n);
  exsum_free_values(v);
  return out;
}

inline void write_values(const std::filesystem::path &path, std::span<const double> values,
                         FileFormat format) {
  detail::check(exsum_write_values(path.c_str(), values.data(), values.size(),
                                   format == FileFormat::bin ? EXSUM_FORMAT_BIN
                                                             : EXSUM_FORMAT_TEXT),
                "write_values");
}

// generator.hpp: GeneratorSpec / generate (generator.cpp:23-45); throws
// std::invalid_argument for n == 0 or odd.
struct GeneratorSpec {
  std::uint64_t n = 0;
  std::uint64_t seed = 1;
  bool permute = false;
};

inline std::vector<double> generate(const GeneratorSpec &spec) {
  if (spec.n == 0 || spec.n % 2 != 0)
    throw std::invalid_argument("generate: n must be a positive even integer");
  std::vector<double> v(spec.n);
  detail::check(exsum_generate(spec.n, spec.seed, spec.permute ? 1 : 0, v.data()), "generate");
  return v;
}

// The B200 path for host-resident arrays: exsum_context (device over PCIe +
// host workers, exact merge).  One sum at a time per context.
class DeviceContext {
 public:
  explicit DeviceContext(int device = 0, std::size_t staging_bytes = std::size_t{256} << 20)
      : c_(exsum_context_create(device, staging_bytes)) {
    if (!c_) throw std::runtime_error("exsum_b200: no CUDA device / context creation failed");
  }
  ~DeviceContext() { exsum_context_free(c_); }
  DeviceContext(const DeviceContext &) = delete;
  DeviceContext &operator=(const DeviceContext &) = delete;

  // exact_sum(values, ExactMethod::large) through the device
  double exact_sum(std::span<const double> values) {
    double out;
    detail::check(exsum_context_sum(c_, values.data(), values.size(), &out, nullptr),
                  "DeviceContext::exact_sum");
    return out;
  }
  double exact_mean(std::span<const double> values) {
    if (values.empty()) throw std::invalid_argument("exact_mean: empty input");
    exsum_partial rec;
    detail::check(exsum_context_sum(c_, values.data(), values.size(), nullptr, &rec),
                  "DeviceContext::exact_mean");
    double out;
    detail::check(exsum_small_mean(&rec.acc, values.size(), &out), "exact_mean");
    return out;
  }
  // one exact_sum per segment values[offsets[i] .. offsets[i+1])
  std::vector<double> exact_sum_segmented(std::span<const double> values,
                                          std::span<const std::uint64_t> offsets) {
    const std::size_t nseg = offsets.empty() ? 0 : offsets.size() - 1;
    std::vector<double> out(nseg);
    detail::check(exsum_context_sum_segmented(c_, values.data(), offsets.data(), nseg,
                                              out.data(), nullptr),
                  "DeviceContext::exact_sum_segmented");
    return out;
  }
  double exact_sum_file(const std::filesystem::path &path, FileFormat format) {
    double out;
    detail::check(exsum_context_sum_file(c_, path.c_str(),
                                         format == FileFormat::bin ? EXSUM_FORMAT_BIN
                                                                   : EXSUM_FORMAT_TEXT,
                                         &out, nullptr, nullptr),
                  "DeviceContext::exact_sum_file");
    return out;
  }
  // host workers beside the device (< 0: all hardware threads, 0: device only)
  void set_host_threads(int threads) {
    detail::check(exsum_context_set_host_threads(c_, threads), "set_host_threads");
  }
  std::pair<std::uint64_t, std::uint64_t> last_split() const {
    std::uint64_t d = 0, h = 0;
    exsum_context_last_split(c_, &d, &h);
    return {d, h};
  }

 private:
  exsum_context *c_;
};

}  // namespace exsum_b200

#endif  // EXSUM_B200_HPP_
