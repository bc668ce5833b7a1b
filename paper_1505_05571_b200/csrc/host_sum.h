// host_sum.h — the library's host superaccumulator workers (see host_sum.cpp).
#ifndef EXSUM_HOST_SUM_H_
#define EXSUM_HOST_SUM_H_

#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <mutex>
#include <thread>
#include <vector>

#include "exsum_b200.h"

namespace exsum_host {

// One worker's exact accumulator: 4096 significand bins (index = sign+exponent,
// as large_accumulator.hpp:99-103) over a 67-chunk small superaccumulator, plus
// the first global index of +Inf / -Inf / NaN.
#ifndef EXSUM_HOST_COPIES
#define EXSUM_HOST_COPIES 1
#endif
struct alignas(64) Acc {
  static constexpr int kCopies = EXSUM_HOST_COPIES;
  static constexpr size_t kBlock = 512;  // terms per blind pass (< 2^10: sentinels cannot wrap)
  uint64_t bin[kCopies][4096];
  int64_t chunk[67];
  uint32_t transfers;
  uint64_t P, M, N, payload;
  uint64_t terms;

  void reset();
  // x[0..n) with global indices gbase .. gbase + n - 1
  void add(const double *x, size_t n, uint64_t gbase);
  // the rounded products a[i] * b[i] (b == a: squares), as sum_products
  // (vector_ops.cpp:72-97) forms them, added like add()
  void add_products(const double *a, const double *b, size_t n, uint64_t gbase);
  // drain the bins; the canonical record with index-resolved Inf/NaN (leaves
  // every bin zero again)
  void finish(exsum_partial *out);
  // One exact_sum of x[b, e) (indices local to the segment) into *out (and
  // *part); the bins must be zero on entry (reset(), or a previous finish()).
  void segment(const double *x, uint64_t b, uint64_t e, double *out, exsum_partial *part);

 private:
  void transfer(uint32_t ix, uint64_t v, uint64_t carry);
  void specials(const uint64_t *b, size_t n, uint64_t gbase);
  void zero_exponents(const uint64_t *b, size_t n);
};

int default_threads();

// Persistent host workers.  A job is a host array and a shared element cursor:
// every worker (the caller is worker 0 in sum(); in the hybrid context sum the
// caller drives the device instead) claims `grain` terms at a time until the
// cursor passes n, so the device feeder and the host workers split the array
// dynamically.  Each worker's record lands in parts()[t].
class Pool {
 public:
  explicit Pool(int nthreads);  // nthreads - 1 helper threads + the caller's slot
  ~Pool();
  Pool(const Pool &) = delete;
  Pool &operator=(const Pool &) = delete;

  bool ok() const;
  int size() const { return static_cast<int>(accs_.size()); }
  // Whole array on the pool, caller included; merged record in *out.  With y:
  // the sum of the rounded products x[i] * y[i] instead.
  void sum(const double *x, size_t n, uint64_t base, exsum_partial *out,
           const double *y = nullptr);
  // Hybrid: helpers start on the shared cursor; the caller does other work,
  // may call run_share(0) itself, then join_helpers().
  void start(const double *x, size_t n, uint64_t base, std::atomic<size_t> *cursor,
             size_t grain, const double *y = nullptr);
  // Hybrid segmented sum: helpers claim `grain` segments at a time from the
  // shared segment cursor and write out[s] (and partials[s]) themselves.
  void start_segments(const double *x, const uint64_t *offs, size_t nseg,
                      std::atomic<size_t> *cursor, size_t grain, double *out,
                      exsum_partial *partials);
  void run_share(int t);
  void join_helpers();
  std::vector<exsum_partial> &parts() { return parts_; }
  uint64_t terms(int t) const { return accs_[static_cast<size_t>(t)]->terms; }

 private:
  struct Job {
    const double *x = nullptr;
    const double *y = nullptr;  // products job: x[i] * y[i]
    size_t n = 0;  // terms, or segments for a segmented job
    uint64_t base = 0;
    std::atomic<size_t> *cursor = nullptr;
    size_t grain = 0;
    const uint64_t *offs = nullptr;  // segmented job: nseg + 1 offsets
    double *out = nullptr;
    exsum_partial *partials = nullptr;
  };
  void run_segments(int t);
  void worker(int t);

  std::vector<Acc *> accs_;
  std::vector<exsum_partial> parts_;
  std::vector<std::thread> threads_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  uint64_t gen_ = 0;
  bool quit_ = false;
  bool failed_ = false;
  std::atomic<int> pending_{0};
  Job job_;
};

}  // namespace exsum_host

#endif  // EXSUM_HOST_SUM_H_
