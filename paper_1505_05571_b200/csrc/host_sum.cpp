// host_sum.cpp — the library's multithreaded HOST exact sum (the CPU side of a
// hybrid host+device sum of a host-resident array).
//
// Why it exists: a reference caller holds its values in host memory
// (exact_sum(std::span<const double>), vector_ops.cpp:121-130).  Shipping them
// to the B200 is capped by PCIe (~55 GB/s H2D on the box), below the 16-thread
// reference (~93 GB/s).  exsum_context_sum therefore streams part of the array
// to the device while these host workers sum the rest, and merges the exact
// partial records (exsum_partial, global Inf/NaN indices) — bits identical to
// exact_sum whatever the split.
//
// The per-term kernel is the paper's large superaccumulator (Neal 2015, §4;
// large_accumulator.hpp:47-59) re-designed for a modern out-of-order core:
//
//   reference: bins of raw bit patterns + an int16 countdown per bin; every
//              add loads, decrements, tests and stores the count (the count
//              both limits overflow and later recovers the implicit ones and
//              strips the exponent bits, large_accumulator.cpp:77-96).
//   here:      bins of SIGNIFICANDS (mantissa | implicit bit, exponent and
//              sign dropped: the bin index carries them), so no count is
//              needed to decode a bin; overflow is caught by the carry flag
//              of the 64-bit add itself (one add < 2^53, so a bin wraps at
//              most once per add and after >= 2048 adds) and the wrapped bin is
//              transferred with its carry bit 2^64 — exact, no countdown.
//   per term:  load, shift, and, or, add-to-memory, never-taken jc.
//
// Zeros and denormals go through the same blind add (their wrongly added
// implicit bits are removed by one counted correction per block); Inf and NaN
// land in two sentinel bins that send their block through a per-term pass
// (first global index, exactly like the device kernels' side channel).
//
// Bins drain into a 67-chunk small superaccumulator (chunk i weighs
// 2^(32 i - 1075), small_accumulator.hpp:27-35) as three 32-bit pieces, the
// reference's transfer geometry (large_accumulator.cpp:81-109) applied to a
// 65-bit significand sum; exsum_core.h canonicalises and rounds.

#include <immintrin.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "exsum_b200.h"
#include "exsum_core.h"
#include "exsum_nvtx.h"
#include "host_sum.h"

using namespace exsum_b200;

namespace exsum_host {

namespace {

constexpr uint64_t kImplicit = uint64_t{1} << kMantBits;
constexpr uint64_t kExpField = uint64_t{0x7FF} << kMantBits;

}  // namespace

void Acc::reset() {
  std::memset(bin, 0, sizeof bin);
  std::memset(chunk, 0, sizeof chunk);
  transfers = 0;
  P = M = N = kNoIndex;
  payload = 0;
  terms = 0;
}

// value = (carry * 2^64 + v) * 2^(e' - 1075), e' = max(e, 1), sign from ix.
// Placed at chunk e' >> 5 shifted by e' & 31: at most 65 + 31 = 96 bits, three
// 32-bit pieces into chunks base .. base + 2 (base + 2 <= 65 < 67).
__attribute__((noinline)) void Acc::transfer(uint32_t ix, uint64_t v, uint64_t carry) {
  const uint32_t e = ix & 0x7FFu;
  const uint32_t ep = e ? e : 1u;
  const uint32_t sh = ep & 31u, base = ep >> 5;
  const unsigned __int128 w = ((static_cast<unsigned __int128>(carry) << 64) | v) << sh;
  const int64_t p0 = static_cast<int64_t>(static_cast<uint64_t>(w) & 0xFFFFFFFFull);
  const int64_t p1 = static_cast<int64_t>(static_cast<uint64_t>(w >> 32) & 0xFFFFFFFFull);
  const int64_t p2 = static_cast<int64_t>(static_cast<uint64_t>(w >> 64));
  if (ix >> 11) {
    chunk[base] -= p0;
    chunk[base + 1] -= p1;
    chunk[base + 2] -= p2;
  } else {
    chunk[base] += p0;
    chunk[base + 1] += p1;
    chunk[base + 2] += p2;
  }
  // each transfer moves < 2^32 into a chunk: canonicalise long before 2^62
  if (++transfers >= (1u << 20)) {
    exsum_canonicalize(chunk);
    transfers = 0;
  }
}

namespace {

// Zero-exponent terms (+-0, denormals) of a block, per sign: they were added
// blindly with an implicit 2^52 each.
struct ZeroExp {
  uint64_t pos, neg;
};

__attribute__((target("avx512f,avx512vpopcntdq"))) ZeroExp zero_exp_avx512(const uint64_t *b,
                                                                            size_t n) {
  const __m512i ef = _mm512_set1_epi64(static_cast<long long>(kExpField));
  const __m512i sg = _mm512_set1_epi64(static_cast<long long>(kSignMask));
  uint64_t pos = 0, neg = 0;
  size_t k = 0;
  for (; k + 8 <= n; k += 8) {
    const __m512i v = _mm512_loadu_si512(b + k);
    const __mmask8 z = _mm512_testn_epi64_mask(v, ef);  // exponent field == 0
    const __mmask8 s = _mm512_test_epi64_mask(v, sg);
    pos += static_cast<uint64_t>(__builtin_popcount(z & static_cast<__mmask8>(~s)));
    neg += static_cast<uint64_t>(__builtin_popcount(z & s));
  }
  for (; k < n; ++k)
    if ((b[k] & kExpField) == 0) (b[k] >> 63 ? neg : pos) += 1;
  return {pos, neg};
}

ZeroExp zero_exp_scalar(const uint64_t *b, size_t n) {
  uint64_t pos = 0, neg = 0;
  for (size_t k = 0; k < n; ++k)
    if ((b[k] & kExpField) == 0) (b[k] >> 63 ? neg : pos) += 1;
  return {pos, neg};
}

const bool kHaveAvx512 =
    __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512vpopcntdq");

}  // namespace

// The block's Inf and NaN (exponent field 0x7FF) after the blind pass put them
// into the sentinel bins 0x7FF / 0xFFF: clear those, record first indices.
__attribute__((noinline)) void Acc::specials(const uint64_t *b, size_t n, uint64_t gbase) {
  for (int c = 0; c < kCopies; ++c) bin[c][0x7FF] = bin[c][0xFFF] = 0;
  for (size_t k = 0; k < n; ++k) {
    const uint64_t v = b[k];
    if ((v & kExpField) != kExpField) continue;
    const uint64_t gi = gbase + k;
    if (v & kMantMask) {
      if (gi < N) {
        N = gi;
        payload = v;
      }
    } else if (v >> 63) {
      if (gi < M) M = gi;
    } else if (gi < P) {
      P = gi;
    }
  }
}

// Implicit bits wrongly added for the block's zero-exponent terms: remove them
// exactly as a transfer of -k 2^52 at exponent 1 (the weight of bins 0x000 /
// 0x800 and of denormals), whatever the bins did meanwhile (carries included).
__attribute__((noinline)) void Acc::zero_exponents(const uint64_t *b, size_t n) {
  const ZeroExp z = kHaveAvx512 ? zero_exp_avx512(b, n) : zero_exp_scalar(b, n);
  if (z.pos) transfer(0x800u, z.pos << kMantBits, 0);  // minus k 2^52 of positive terms
  if (z.neg) transfer(0x000u, z.neg << kMantBits, 0);  // plus k 2^52 of negative terms
}

#ifndef EXSUM_HOST_PREFETCH
#define EXSUM_HOST_PREFETCH 512  // software prefetch distance in terms (4 KB; 0: hardware only)
#endif

// Blind pass: every term's significand (mantissa | implicit bit) is added to
// bin copy (k mod kCopies) of its sign+exponent index — no per-term test for
// zeros, denormals or specials.  Afterwards, once per block:
//   * bins 0x000 / 0x800 changed -> the block held zero-exponent terms: the
//     wrongly added implicit bits are removed by a counted correction
//     (zero_exponents; the denormals' mantissas are already in the right bin);
//   * sentinel bins 0x7FF / 0xFFF nonzero -> Inf/NaN in the block (specials);
//     they hold nothing else, and a block of <= 2^10 terms cannot wrap them.
// The copies break the store-to-load chain when consecutive terms share an
// exponent (U[0,1): half the terms in one bin).
void Acc::add(const double *x, size_t n, uint64_t gbase) {
  const uint64_t *b = reinterpret_cast<const uint64_t *>(x);
  size_t i = 0;
  while (i < n) {
    const size_t len = n - i < kBlock ? n - i : kBlock;
    const uint64_t *blk = b + i;
    uint64_t z0[kCopies], z8[kCopies];
    for (int c = 0; c < kCopies; ++c) {
      z0[c] = bin[c][0];
      z8[c] = bin[c][0x800];
    }
    size_t k = 0;
    for (; k + 8 <= len; k += 8) {
#if EXSUM_HOST_PREFETCH
      __builtin_prefetch(blk + k + EXSUM_HOST_PREFETCH, 0, 0);
#endif
#pragma GCC unroll 8
      for (int j = 0; j < 8; ++j) {
        const int c = j % kCopies;
        const uint64_t v = blk[k + j];
        const uint64_t ix = v >> kMantBits;
        uint64_t s;
        if (__builtin_expect(
                __builtin_add_overflow(bin[c][ix], (v & kMantMask) | kImplicit, &s), 0)) {
          transfer(static_cast<uint32_t>(ix), s, 1);
          s = 0;
        }
        bin[c][ix] = s;
      }
    }
    for (; k < len; ++k) {
      const uint64_t v = blk[k];
      const uint64_t ix = v >> kMantBits;
      uint64_t s;
      if (__builtin_add_overflow(bin[0][ix], (v & kMantMask) | kImplicit, &s)) {
        transfer(static_cast<uint32_t>(ix), s, 1);
        s = 0;
      }
      bin[0][ix] = s;
    }
    uint64_t zchg = 0, sentinel = 0;
    for (int c = 0; c < kCopies; ++c) {
      zchg |= (bin[c][0] ^ z0[c]) | (bin[c][0x800] ^ z8[c]);
      sentinel |= bin[c][0x7FF] | bin[c][0xFFF];
    }
    if (__builtin_expect(zchg != 0, 0)) zero_exponents(blk, len);
    if (__builtin_expect(sentinel != 0, 0)) specials(blk, len, gbase + i);
    i += len;
  }
  terms += n;
}

// Products in blocks of 512 (rounded by the host multiply, baseline x86-64 SSE2,
// no FMA contraction: the reference's a[i] * b[i] bit for bit, NaN and 0 * Inf
// rules included), then the blind-add pass over the block.
// The operand order matters for NaN payloads (x86 returns the FIRST operand's
// NaN, quieted, when both are NaN), and a compiler may commute a plain a * b:
// the multiply is pinned as mulsd with a as the destination operand.
static inline double x86_mul(double a, double b) {
#if defined(__x86_64__) || defined(__i386__)
  __asm__("mulsd %1, %0" : "+x"(a) : "x"(b));
  return a;
#else
  return a * b;
#endif
}

void Acc::add_products(const double *a, const double *b, size_t n, uint64_t gbase) {
  double prod[kBlock];
  for (size_t i = 0; i < n; i += kBlock) {
    const size_t len = n - i < kBlock ? n - i : kBlock;
    for (size_t k = 0; k < len; ++k) prod[k] = x86_mul(a[i + k], b[i + k]);
    add(prod, len, gbase + i);
  }
}

void Acc::finish(exsum_partial *out) {
  for (int c = 0; c < kCopies; ++c)
    for (uint32_t g = 0; g < 4096; g += 8) {
      uint64_t any = 0;
      for (int k = 0; k < 8; ++k) any |= bin[c][g + k];
      if (!any) continue;  // most groups are empty for narrow data
      for (uint32_t ix = g; ix < g + 8; ++ix)
        if (bin[c][ix]) {
          transfer(ix, bin[c][ix], 0);
          bin[c][ix] = 0;
        }
    }
  std::memset(out, 0, sizeof *out);
  std::memcpy(out->acc.chunk, chunk, sizeof chunk);
  exsum_canonicalize(out->acc.chunk);
  exsum_resolve_specials(P, M, N, payload, &out->acc.inf_bits, &out->acc.nan_bits);
  out->acc.adds_until_propagate = kCarryTerms;
  out->first_pos_inf = P;
  out->first_neg_inf = M;
  out->first_nan = N;
  out->nan_payload = payload;
}

void Acc::segment(const double *x, uint64_t b, uint64_t e, double *out, exsum_partial *part) {
  std::memset(chunk, 0, sizeof chunk);
  transfers = 0;
  P = M = N = kNoIndex;
  payload = 0;
  if (e > b) add(x + b, e - b, 0);
  exsum_partial rec;
  finish(&rec);
  if (part) *part = rec;
  exsum_partial_round(&rec, out);
}

int default_threads() {
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? static_cast<int>(hc) : 1;
}

// ------------------------------------------------------------------ Pool

// No exception leaves the pool (it is built behind the C ABI): an allocation or
// thread-creation failure leaves ok() false; the threads already started are
// joined by the destructor.
Pool::Pool(int nthreads) {
  if (nthreads < 1) nthreads = 1;
  try {
    accs_.resize(static_cast<size_t>(nthreads), nullptr);
    for (auto &a : accs_) a = new (std::nothrow) Acc;
    parts_.reserve(static_cast<size_t>(nthreads));
    for (int t = 1; t < nthreads; ++t) threads_.emplace_back([this, t] { worker(t); });
  } catch (...) {
    failed_ = true;
  }
}

Pool::~Pool() {
  {
    std::lock_guard<std::mutex> lk(m_);
    quit_ = true;
    ++gen_;
  }
  cv_.notify_all();
  for (auto &th : threads_) th.join();
  for (auto *a : accs_) delete a;
}

bool Pool::ok() const {
  if (failed_ || accs_.empty()) return false;
  for (auto *a : accs_)
    if (!a) return false;
  return true;
}

void Pool::run_segments(int t) {
  EXSUM_NVTX("exsum_host: worker segments");
  Acc *a = accs_[static_cast<size_t>(t)];
  a->reset();
  for (;;) {
    const size_t s0 = job_.cursor->fetch_add(job_.grain, std::memory_order_relaxed);
    if (s0 >= job_.n) break;
    const size_t s1 = job_.n - s0 < job_.grain ? job_.n : s0 + job_.grain;
    for (size_t s = s0; s < s1; ++s) {
      const uint64_t b = job_.offs[s], e = job_.offs[s + 1];
      a->segment(job_.x, b, e < b ? b : e, job_.out + s, job_.partials ? job_.partials + s : nullptr);
    }
  }
}

void Pool::run_share(int t) {
  if (job_.offs) {
    run_segments(t);
    return;
  }
  EXSUM_NVTX("exsum_host: worker share");
  Acc *a = accs_[static_cast<size_t>(t)];
  a->reset();
  for (;;) {
    const size_t begin = job_.cursor->fetch_add(job_.grain, std::memory_order_relaxed);
    if (begin >= job_.n) break;
    const size_t len = job_.n - begin < job_.grain ? job_.n - begin : job_.grain;
    if (job_.y)
      a->add_products(job_.x + begin, job_.y + begin, len, job_.base + begin);
    else
      a->add(job_.x + begin, len, job_.base + begin);
  }
  a->finish(&parts_[static_cast<size_t>(t)]);
}

void Pool::worker(int t) {
  uint64_t seen = 0;
  for (;;) {
    {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (quit_) return;
    }
    run_share(t);
    if (pending_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
      std::lock_guard<std::mutex> lk(m_);
      done_cv_.notify_all();
    }
  }
}

void Pool::start(const double *x, size_t n, uint64_t base, std::atomic<size_t> *cursor,
                 size_t grain, const double *y) {
  exsum_partial empty{};
  empty.acc.adds_until_propagate = kCarryTerms;
  empty.first_pos_inf = empty.first_neg_inf = empty.first_nan = kNoIndex;
  parts_.assign(accs_.size(), empty);
  Job j;
  j.x = x;
  j.y = y;
  j.n = n;
  j.base = base;
  j.cursor = cursor;
  j.grain = grain ? grain : (size_t{1} << 18);
  job_ = j;
  pending_.store(static_cast<int>(threads_.size()), std::memory_order_relaxed);
  {
    std::lock_guard<std::mutex> lk(m_);
    ++gen_;
  }
  cv_.notify_all();
}

void Pool::start_segments(const double *x, const uint64_t *offs, size_t nseg,
                          std::atomic<size_t> *cursor, size_t grain, double *out,
                          exsum_partial *partials) {
  Job j;
  j.x = x;
  j.n = nseg;
  j.cursor = cursor;
  j.grain = grain ? grain : 4;
  j.offs = offs;
  j.out = out;
  j.partials = partials;
  job_ = j;
  pending_.store(static_cast<int>(threads_.size()), std::memory_order_relaxed);
  {
    std::lock_guard<std::mutex> lk(m_);
    ++gen_;
  }
  cv_.notify_all();
}

void Pool::join_helpers() {
  std::unique_lock<std::mutex> lk(m_);
  done_cv_.wait(lk, [&] { return pending_.load(std::memory_order_acquire) == 0; });
}

void Pool::sum(const double *x, size_t n, uint64_t base, exsum_partial *out, const double *y) {
  std::atomic<size_t> cursor{0};
  start(x, n, base, &cursor, 0, y);
  run_share(0);  // the calling thread is worker 0
  join_helpers();
  exsum_partial_merge(parts_.data(), parts_.size(), out, nullptr);
}

}  // namespace exsum_host

// ================================================================== C ABI

extern "C" int exsum_host_sum(const double *x, size_t n, uint64_t base_index, int threads,
                              double *result, exsum_partial *partial) {
  EXSUM_NVTX("exsum_host_sum");
  if ((n && !x) || (!result && !partial)) return EXSUM_EINVAL;
  if (threads <= 0) threads = exsum_host::default_threads();
  // no more threads than 1 Mi-term shares: thread start-up would dominate
  const size_t cap = n >> 20;
  if (static_cast<size_t>(threads) > cap) threads = cap ? static_cast<int>(cap) : 1;
  exsum_partial rec;
  if (threads == 1) {
    exsum_host::Acc *a = new (std::nothrow) exsum_host::Acc;
    if (!a) return EXSUM_ENOMEM;
    a->reset();
    a->add(x, n, base_index);
    a->finish(&rec);
    delete a;
  } else {
    exsum_host::Pool pool(threads);
    if (!pool.ok()) return EXSUM_ENOMEM;
    pool.sum(x, n, base_index, &rec);
  }
  if (partial) *partial = rec;
  if (result) exsum_partial_round(&rec, result);
  return EXSUM_OK;
}

// exact_sum(values, ExactMethod) on the host (vector_ops.cpp:121-130), one call:
// method 0 = small (SmallAccumulator add(span) + round, exsum_small_*),
// method 1 = large (this file's host kernel on the calling thread; the same bits
// as LargeAccumulator + round).
extern "C" int exsum_exact_sum(const double *x, size_t n, int method, double *out) {
  if (!out || (n && !x) || (method != 0 && method != 1)) return EXSUM_EINVAL;
  if (method == 0) {
    exsum_small acc;
    exsum_small_init(&acc);
    exsum_small_add_array(&acc, x, n);
    return exsum_small_round(&acc, out);
  }
  try {
    thread_local exsum_host::Acc *acc = nullptr;  // 32 KB of bins, reused per thread
    if (!acc && !(acc = new (std::nothrow) exsum_host::Acc)) return EXSUM_ENOMEM;
    exsum_partial rec;
    acc->reset();
    acc->add(x, n, 0);
    acc->finish(&rec);
    return exsum_partial_round(&rec, out);
  } catch (...) {
    return EXSUM_ENOMEM;
  }
}

// sum_products on the host: sqnorm (b == a) / dot (vector_ops.cpp:72-97,143-155);
// threads <= 0: every hardware thread, capped at one per 2^20 products.
extern "C" int exsum_host_products(const double *a, const double *b, size_t n, int threads,
                                   double *out) {
  EXSUM_NVTX("exsum_host_products");
  if (!out || (n && (!a || !b))) return EXSUM_EINVAL;
  if (threads <= 0) threads = exsum_host::default_threads();
  const size_t cap = n >> 20;
  if (static_cast<size_t>(threads) > cap) threads = cap ? static_cast<int>(cap) : 1;
  try {
    exsum_partial rec;
    if (threads == 1) {
      thread_local exsum_host::Acc *acc = nullptr;
      if (!acc && !(acc = new (std::nothrow) exsum_host::Acc)) return EXSUM_ENOMEM;
      acc->reset();
      acc->add_products(a, b, n, 0);
      acc->finish(&rec);
    } else {
      exsum_host::Pool pool(threads);
      if (!pool.ok()) return EXSUM_ENOMEM;
      pool.sum(a, n, 0, &rec, b);
    }
    return exsum_partial_round(&rec, out);
  } catch (...) {
    return EXSUM_ENOMEM;
  }
}
