// context.cu — exact sum of a HOST array: the B200 and the host cores together.
//
// exsum_context_sum is the drop-in for exact_sum(values, ExactMethod::large)
// (vector_ops.cpp:121-130) when the caller's values live in host memory, as
// they do for every reference caller.  The array is split DYNAMICALLY between
//
//   * the device feeder (the calling thread): claims chunks from a shared
//     cursor, copies each host->device over PCIe into a 4-slot device staging
//     ring (copy stream) and accumulates it there (exsum_cuda_accumulate with the
//     chunk's global base index, compute stream); at most three chunks in
//     flight, so the DMA engine never idles and the device never hoards work;
//   * the host workers (exsum_host::Pool, host_sum.cpp): claim small chunks
//     from the same cursor and sum them with the library's own host kernel.
//
// Each side ends with an exact exsum_partial record (global Inf/NaN indices);
// exsum_partial_merge combines them, so the bits equal exact_sum(values) for
// any split.  Why both: PCIe caps the device at ~55 GB/s H2D, below what the
// host cores stream; the device adds its PCIe rate on top of the cores'.
// Pinned host memory is DMA'd directly; pageable memory is staged by the feeder
// through pinned bounce buffers.  exsum_context_set_host_threads(ctx, 0) gives a
// device-only sum (the PCIe-bound path).

#include <cuda_runtime.h>
#include <fcntl.h>
#include <stdint.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <new>
#include <string>

#include "exsum_b200.h"
#include "exsum_nvtx.h"
#include "host_sum.h"

namespace {
constexpr int kSlots = 4;     // device staging buffers
constexpr int kInFlight = 3;  // chunks claimed by the feeder and not yet copied (DMA queue
                              // depth: covers the feeder's wake-up latency among busy workers)
constexpr size_t kHostGrain = size_t{1} << 18;  // terms per host-worker claim (2 MB)
// Below this many terms a host array is summed by the calling thread alone: the
// device round trip (~35 us: copy, accumulate, finalize, readback) and a worker
// wake-up cost more than the whole sum on one core (profiles/r02_latency_probe.log:
// 1e3 / 1e4 / 1e5 terms: device 37 / 49 / 99 us, one core 4 / 8 / 46 us).
// exsum_context_set_host_threads(ctx, 0) keeps every size on the device.
constexpr size_t kHostOnlyTerms = size_t{1} << 17;
}  // namespace

struct exsum_context {
  int device = 0;
  mutable std::mutex busy;  // one sum at a time per context (staging, workspace, pool)
  void *ws = nullptr;
  size_t ws_bytes = 0;
  double *stage[kSlots] = {};
  size_t stage_elems = 0;
  cudaStream_t copy = nullptr, compute = nullptr;
  cudaEvent_t copied[kSlots] = {}, consumed[kSlots] = {};
  double *d_result = nullptr;
  exsum_partial *d_partial = nullptr;
  exsum_partial *h_partial = nullptr;  // pinned landing slot of the device record
  double *host[kSlots] = {};           // pinned bounce buffers (pageable input, files)
  int host_threads = -1;               // < 0: all hardware threads; 0: device only
  exsum_host::Pool *pool = nullptr;
  exsum_host::Acc *small = nullptr;  // the calling thread's accumulator for small arrays
  uint64_t last_device_terms = 0, last_host_terms = 0;
  // segmented sums of host arrays (allocated on first use)
  void *seg_ws = nullptr;
  size_t seg_ws_bytes = 0;
  uint64_t *d_offs[kSlots] = {}, *h_offs[kSlots] = {};
  double *d_out[kSlots] = {}, *h_out[kSlots] = {};
  exsum_partial *d_parts[kSlots] = {}, *h_parts[kSlots] = {};
};

namespace {

void destroy(exsum_context *c) {
  if (!c) return;
  delete c->pool;
  delete c->small;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  for (int i = 0; i < kSlots; ++i) {
    if (c->host[i]) cudaFreeHost(c->host[i]);
    if (c->stage[i]) cudaFree(c->stage[i]);
    if (c->copied[i]) cudaEventDestroy(c->copied[i]);
    if (c->consumed[i]) cudaEventDestroy(c->consumed[i]);
  }
  if (c->h_partial) cudaFreeHost(c->h_partial);
  for (int i = 0; i < kSlots; ++i) {
    if (c->d_offs[i]) cudaFree(c->d_offs[i]);
    if (c->d_out[i]) cudaFree(c->d_out[i]);
    if (c->d_parts[i]) cudaFree(c->d_parts[i]);
    if (c->h_offs[i]) cudaFreeHost(c->h_offs[i]);
    if (c->h_out[i]) cudaFreeHost(c->h_out[i]);
    if (c->h_parts[i]) cudaFreeHost(c->h_parts[i]);
  }
  if (c->seg_ws) cudaFree(c->seg_ws);
  if (c->ws) cudaFree(c->ws);
  if (c->d_result) cudaFree(c->d_result);
  if (c->d_partial) cudaFree(c->d_partial);
  if (c->copy) cudaStreamDestroy(c->copy);
  if (c->compute) cudaStreamDestroy(c->compute);
  cudaSetDevice(prev);
  delete c;
}

int ensure_bounce(exsum_context *c) {
  for (int i = 0; i < kSlots; ++i)
    if (!c->host[i] && cudaMallocHost(&c->host[i], c->stage_elems * sizeof(double)) != cudaSuccess)
      return EXSUM_ECUDA;
  return EXSUM_OK;
}

// After a failed sum the workspace may hold part of an accumulation: clear it so
// the next sum on this context starts from zero (drain both streams first).
void reset_after_error(exsum_context *c) {
  cudaGetLastError();
  cudaStreamSynchronize(c->copy);
  cudaStreamSynchronize(c->compute);
  exsum_cuda_workspace_init(c->ws, c->ws_bytes, c->compute);
  if (c->seg_ws) exsum_cuda_workspace_init(c->seg_ws, c->seg_ws_bytes, c->compute);
  cudaStreamSynchronize(c->compute);
}

constexpr size_t kGroupSegs = 16384;  // segments per device group (segmented sums)

int ensure_segmented(exsum_context *c, bool partials) {
  if (!c->seg_ws) {
    c->seg_ws_bytes = exsum_cuda_segmented_workspace_bytes(kGroupSegs);
    if (cudaMalloc(&c->seg_ws, c->seg_ws_bytes) != cudaSuccess) {
      c->seg_ws = nullptr;
      return EXSUM_ENOMEM;
    }
    if (exsum_cuda_workspace_init(c->seg_ws, c->seg_ws_bytes, c->compute) != EXSUM_OK ||
        cudaStreamSynchronize(c->compute) != cudaSuccess)
      return EXSUM_ECUDA;
  }
  for (int i = 0; i < kSlots; ++i) {
    if (!c->d_offs[i] &&
        (cudaMalloc(&c->d_offs[i], (kGroupSegs + 1) * 8) != cudaSuccess ||
         cudaMalloc(&c->d_out[i], kGroupSegs * 8) != cudaSuccess ||
         cudaMallocHost(&c->h_offs[i], (kGroupSegs + 1) * 8) != cudaSuccess ||
         cudaMallocHost(&c->h_out[i], kGroupSegs * 8) != cudaSuccess))
      return EXSUM_ENOMEM;
    if (partials && !c->d_parts[i] &&
        (cudaMalloc(&c->d_parts[i], kGroupSegs * sizeof(exsum_partial)) != cudaSuccess ||
         cudaMallocHost(&c->h_parts[i], kGroupSegs * sizeof(exsum_partial)) != cudaSuccess))
      return EXSUM_ENOMEM;
  }
  return EXSUM_OK;
}

bool is_pinned(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Device feeder: claim chunks from *cursor until it passes n; copy + accumulate.
// Returns the number of terms it took, or sets *st.
uint64_t feed_device(exsum_context *c, const double *h_x, size_t n, uint64_t base,
                     std::atomic<size_t> *cursor, bool pinned, bool hybrid, int *st) {
  EXSUM_NVTX("exsum_context: device feed");
  uint64_t taken = 0;
  for (int i = 0;; ++i) {
    const int b = i % kSlots;
    if (i >= kInFlight && cudaEventSynchronize(c->copied[(i - kInFlight) % kSlots]) != cudaSuccess) {
      *st = EXSUM_ECUDA;
      break;
    }
    // guided claim: no more than a quarter of what is left while the host shares
    const size_t seen = cursor->load(std::memory_order_relaxed);
    if (seen >= n) break;
    size_t want = c->stage_elems;
    if (hybrid) want = std::min(want, std::max<size_t>((n - seen) / 4, size_t{1} << 16));
    const size_t off = cursor->fetch_add(want, std::memory_order_relaxed);
    if (off >= n) break;
    const size_t len = std::min(want, n - off);
    const double *src = h_x + off;
    if (!pinned) {  // bounce b is free: its last copy (chunk i - kSlots) completed above
      memcpy(c->host[b], src, len * sizeof(double));
      src = c->host[b];
    }
    if ((i >= kSlots && cudaStreamWaitEvent(c->copy, c->consumed[b], 0) != cudaSuccess) ||
        cudaMemcpyAsync(c->stage[b], src, len * sizeof(double), cudaMemcpyHostToDevice,
                        c->copy) != cudaSuccess ||
        cudaEventRecord(c->copied[b], c->copy) != cudaSuccess ||
        cudaStreamWaitEvent(c->compute, c->copied[b], 0) != cudaSuccess) {
      *st = EXSUM_ECUDA;
      break;
    }
    *st = exsum_cuda_accumulate(c->stage[b], len, base + off, c->ws, c->ws_bytes, c->compute);
    if (*st != EXSUM_OK) break;
    if (cudaEventRecord(c->consumed[b], c->compute) != cudaSuccess) {
      *st = EXSUM_ECUDA;
      break;
    }
    taken += len;
  }
  return taken;
}

}  // namespace

extern "C" {

exsum_context *exsum_context_create(int device, size_t staging_bytes) {
  if (staging_bytes < (size_t{3} << 20)) staging_bytes = size_t{3} << 20;
  exsum_context *c = new (std::nothrow) exsum_context;
  if (!c) return nullptr;
  c->device = device;
  int prev = 0;
  cudaGetDevice(&prev);
  bool ok = cudaSetDevice(device) == cudaSuccess;
  // one device chunk: a third of the staging bytes, capped at 64 MB (PCIe runs at
  // full rate from a few MB; smaller chunks balance better against the host)
  c->stage_elems = std::min(staging_bytes / kSlots, size_t{64} << 20) / sizeof(double);
  c->stage_elems &= ~size_t{3};
  c->ws_bytes = exsum_cuda_workspace_bytes();
  ok = ok && cudaMalloc(&c->ws, c->ws_bytes) == cudaSuccess;
  ok = ok && cudaMalloc(&c->d_result, sizeof(double)) == cudaSuccess;
  ok = ok && cudaMalloc(&c->d_partial, sizeof(exsum_partial)) == cudaSuccess;
  ok = ok && cudaMallocHost(&c->h_partial, sizeof(exsum_partial)) == cudaSuccess;
  for (int i = 0; i < kSlots && ok; ++i) {
    ok = cudaMalloc(&c->stage[i], c->stage_elems * sizeof(double)) == cudaSuccess;
    // blocking-sync events: the feeder sleeps while DMA runs, leaving its core to
    // the host workers
    ok = ok && cudaEventCreateWithFlags(&c->copied[i], cudaEventDisableTiming |
                                                           cudaEventBlockingSync) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->consumed[i], cudaEventDisableTiming) == cudaSuccess;
  }
  ok = ok && cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&c->compute, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && exsum_cuda_workspace_init(c->ws, c->ws_bytes, c->compute) == EXSUM_OK;
  ok = ok && cudaStreamSynchronize(c->compute) == cudaSuccess;
  cudaSetDevice(prev);
  if (!ok) {
    destroy(c);
    return nullptr;
  }
  return c;
}

void exsum_context_free(exsum_context *ctx) { destroy(ctx); }

int exsum_context_set_host_threads(exsum_context *c, int threads) {
  if (!c) return EXSUM_EINVAL;
  std::lock_guard<std::mutex> lk(c->busy);
  if (threads != c->host_threads) {
    delete c->pool;
    c->pool = nullptr;
    c->host_threads = threads;
  }
  return EXSUM_OK;
}

int exsum_context_last_split(const exsum_context *c, uint64_t *device_terms,
                             uint64_t *host_terms) {
  if (!c) return EXSUM_EINVAL;
  std::lock_guard<std::mutex> lk(c->busy);
  if (device_terms) *device_terms = c->last_device_terms;
  if (host_terms) *host_terms = c->last_host_terms;
  return EXSUM_OK;
}

int exsum_context_sum(exsum_context *c, const double *h_x, size_t n, double *h_result,
                      exsum_partial *h_partial) {
  return exsum_context_sum_at(c, h_x, n, 0, h_result, h_partial);
}

int exsum_context_sum_at(exsum_context *c, const double *h_x, size_t n, uint64_t base_index,
                         double *h_result, exsum_partial *h_partial) {
  EXSUM_NVTX("exsum_context_sum");
  if (!c || (n && !h_x) || (!h_result && !h_partial)) return EXSUM_EINVAL;
  std::lock_guard<std::mutex> lk(c->busy);
  if (n < kHostOnlyTerms && c->host_threads != 0) {
    if (!c->small && !(c->small = new (std::nothrow) exsum_host::Acc)) return EXSUM_ENOMEM;
    exsum_partial rec;
    c->small->reset();
    c->small->add(h_x, n, base_index);
    c->small->finish(&rec);
    if (h_partial) *h_partial = rec;
    if (h_result) exsum_partial_round(&rec, h_result);
    c->last_device_terms = 0;
    c->last_host_terms = n;
    return EXSUM_OK;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(c->device) != cudaSuccess) return EXSUM_ECUDA;
  const bool pinned = n == 0 || is_pinned(h_x);
  int st = pinned ? EXSUM_OK : ensure_bounce(c);
  // host workers: every hardware thread by default (the feeder mostly sleeps in
  // blocking event waits)
  int workers = c->host_threads < 0 ? exsum_host::default_threads() : c->host_threads;
  if (st == EXSUM_OK && workers > 0 && (!c->pool || c->pool->size() != workers + 1)) {
    delete c->pool;
    c->pool = new (std::nothrow) exsum_host::Pool(workers + 1);  // slot 0: the feeder
    if (!c->pool || !c->pool->ok()) {
      delete c->pool;
      c->pool = nullptr;
      workers = 0;
    }
  }
  std::atomic<size_t> cursor{0};
  const bool hybrid = workers > 0 && c->pool;
  if (st == EXSUM_OK && hybrid) c->pool->start(h_x, n, base_index, &cursor, kHostGrain);
  uint64_t dev_terms = 0;
  if (st == EXSUM_OK) dev_terms = feed_device(c, h_x, n, base_index, &cursor, pinned, hybrid, &st);
  // the device's record (skipped when the host workers left it nothing)
  const bool dev_part = dev_terms > 0 || !hybrid;
  if (st == EXSUM_OK && dev_part)
    st = exsum_cuda_finalize(c->d_result, c->d_partial, c->ws, c->ws_bytes, c->compute);
  if (st == EXSUM_OK && dev_part &&
      cudaMemcpyAsync(c->h_partial, c->d_partial, sizeof(exsum_partial), cudaMemcpyDeviceToHost,
                      c->compute) != cudaSuccess)
    st = EXSUM_ECUDA;
  if (cudaStreamSynchronize(c->compute) != cudaSuccess && st == EXSUM_OK) st = EXSUM_ECUDA;
  if (hybrid) c->pool->join_helpers();  // workers finish the array even if the device failed
  if (st != EXSUM_OK) {
    reset_after_error(c);
  } else {
    exsum_partial merged;
    if (hybrid) {
      auto &parts = c->pool->parts();
      if (dev_part) parts[0] = *c->h_partial;  // else parts[0] is the empty record
      exsum_partial_merge(parts.data(), parts.size(), &merged, nullptr);
    } else {
      merged = *c->h_partial;
    }
    if (h_partial) *h_partial = merged;
    if (h_result) exsum_partial_round(&merged, h_result);
    c->last_device_terms = dev_terms;
    c->last_host_terms = n - dev_terms;
  }
  cudaSetDevice(prev);
  return st;
}


int exsum_context_sum_segmented(exsum_context *c, const double *h_x, const uint64_t *h_offsets,
                                size_t nseg, double *h_out, exsum_partial *h_partials) {
  EXSUM_NVTX("exsum_context_sum_segmented");
  if (!c || (nseg && (!h_offsets || !h_out))) return EXSUM_EINVAL;
  if (nseg == 0) return EXSUM_OK;
  // the span of values the segments touch (offsets need not be monotonic: a
  // decreasing pair is an empty segment)
  uint64_t lo = h_offsets[0], hi = h_offsets[0];
  for (size_t s = 1; s <= nseg; ++s) {
    lo = h_offsets[s] < lo ? h_offsets[s] : lo;
    hi = h_offsets[s] > hi ? h_offsets[s] : hi;
  }
  if (hi > lo && !h_x) return EXSUM_EINVAL;
  std::lock_guard<std::mutex> lk(c->busy);
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(c->device) != cudaSuccess) return EXSUM_ECUDA;
  const bool pinned = hi == lo || is_pinned(h_x + lo);
  int st = ensure_segmented(c, h_partials != nullptr);
  if (st == EXSUM_OK && !pinned) st = ensure_bounce(c);
  int workers = c->host_threads < 0 ? exsum_host::default_threads() : c->host_threads;
  if (st == EXSUM_OK && hi - lo < kHostOnlyTerms && c->host_threads != 0) {
    // a small segment list: the calling thread alone (see kHostOnlyTerms)
    if (!c->small && !(c->small = new (std::nothrow) exsum_host::Acc)) st = EXSUM_ENOMEM;
    if (st == EXSUM_OK) {
      c->small->reset();
      uint64_t total = 0;
      for (size_t s = 0; s < nseg; ++s) {
        const uint64_t b = h_offsets[s], e = h_offsets[s + 1];
        c->small->segment(h_x, b, e < b ? b : e, h_out + s, h_partials ? h_partials + s : nullptr);
        total += e > b ? e - b : 0;
      }
      c->last_device_terms = 0;
      c->last_host_terms = total;
    }
    cudaSetDevice(prev);
    return st;
  }
  if (st == EXSUM_OK && workers > 0 && (!c->pool || c->pool->size() != workers + 1)) {
    delete c->pool;
    c->pool = new (std::nothrow) exsum_host::Pool(workers + 1);
    if (!c->pool || !c->pool->ok()) {
      delete c->pool;
      c->pool = nullptr;
      workers = 0;
    }
  }
  const bool hybrid = workers > 0 && c->pool;
  std::atomic<size_t> cursor{0};
  if (st == EXSUM_OK && hybrid)
    c->pool->start_segments(h_x, h_offsets, nseg, &cursor, 4, h_out, h_partials);
  // device feeder: groups of whole segments, each group's value span <= one chunk
  size_t pend0[kSlots] = {}, pend1[kSlots] = {};
  bool pending[kSlots] = {};
  uint64_t dev_terms = 0;
  auto drain_slot = [&](int b) {
    if (!pending[b]) return true;
    if (cudaEventSynchronize(c->consumed[b]) != cudaSuccess) return false;
    memcpy(h_out + pend0[b], c->h_out[b], (pend1[b] - pend0[b]) * 8);
    if (h_partials)
      memcpy(h_partials + pend0[b], c->h_parts[b], (pend1[b] - pend0[b]) * sizeof(exsum_partial));
    pending[b] = false;
    return true;
  };
  for (int i = 0; st == EXSUM_OK; ++i) {
    const int b = i % kSlots;
    if (i >= kInFlight && cudaEventSynchronize(c->copied[(i - kInFlight) % kSlots]) != cudaSuccess) {
      st = EXSUM_ECUDA;
      break;
    }
    if (!drain_slot(b)) {
      st = EXSUM_ECUDA;
      break;
    }
    // claim [s0, s1): as many segments as fit one staging chunk (CAS: host
    // workers move the same cursor with fetch_add)
    size_t s0 = cursor.load(std::memory_order_relaxed), s1 = 0;
    uint64_t glo = 0, ghi = 0;
    bool got = false, longseg = false;
    while (s0 < nseg) {
      glo = ghi = h_offsets[s0];
      s1 = s0;
      while (s1 < nseg && s1 - s0 < kGroupSegs) {
        const uint64_t nlo = h_offsets[s1 + 1] < glo ? h_offsets[s1 + 1] : glo;
        const uint64_t nhi = h_offsets[s1 + 1] > ghi ? h_offsets[s1 + 1] : ghi;
        if (nhi - nlo > c->stage_elems) break;
        glo = nlo;
        ghi = nhi;
        ++s1;
      }
      longseg = s1 == s0;  // one segment larger than a chunk: streamed on its own
      if (longseg) s1 = s0 + 1;
      if (cursor.compare_exchange_weak(s0, s1, std::memory_order_relaxed)) {
        got = true;
        break;
      }
    }
    if (!got) break;
    if (longseg) {
      // the ring's pending groups first, then the segment through the incremental
      // path (chunked copies + exsum_cuda_accumulate, local indices) and a finalize
      for (int k = 0; k < kSlots && st == EXSUM_OK; ++k)
        if (!drain_slot(k)) st = EXSUM_ECUDA;
      if (st != EXSUM_OK) break;
      const uint64_t b0 = h_offsets[s0], e0 = h_offsets[s0 + 1];
      std::atomic<size_t> sub{0};
      dev_terms += feed_device(c, h_x + b0, e0 - b0, 0, &sub, is_pinned(h_x + b0), false, &st);
      if (st == EXSUM_OK)
        st = exsum_cuda_finalize(c->d_result, c->d_partial, c->ws, c->ws_bytes, c->compute);
      if (st == EXSUM_OK &&
          (cudaMemcpyAsync(c->h_partial, c->d_partial, sizeof(exsum_partial),
                           cudaMemcpyDeviceToHost, c->compute) != cudaSuccess ||
           cudaStreamSynchronize(c->compute) != cudaSuccess))
        st = EXSUM_ECUDA;
      if (st != EXSUM_OK) break;
      if (h_partials) h_partials[s0] = *c->h_partial;
      exsum_partial_round(c->h_partial, h_out + s0);
      i = -1;  // the ring restarts empty
      continue;
    }
    const size_t len = ghi - glo, ns = s1 - s0;
    const double *src = h_x + glo;
    if (!pinned && len) {
      memcpy(c->host[b], src, len * sizeof(double));
      src = c->host[b];
    }
    memcpy(c->h_offs[b], h_offsets + s0, (ns + 1) * 8);
    if ((i >= kSlots && cudaStreamWaitEvent(c->copy, c->consumed[b], 0) != cudaSuccess) ||
        (len && cudaMemcpyAsync(c->stage[b], src, len * sizeof(double), cudaMemcpyHostToDevice,
                                c->copy) != cudaSuccess) ||
        cudaMemcpyAsync(c->d_offs[b], c->h_offs[b], (ns + 1) * 8, cudaMemcpyHostToDevice,
                        c->copy) != cudaSuccess ||
        cudaEventRecord(c->copied[b], c->copy) != cudaSuccess ||
        cudaStreamWaitEvent(c->compute, c->copied[b], 0) != cudaSuccess) {
      st = EXSUM_ECUDA;
      break;
    }
    // the kernel addresses x + offs[s]: hand it the staged span shifted back by glo
    st = exsum_cuda_sum_segmented(c->stage[b] - glo, c->d_offs[b], ns, c->d_out[b],
                                  h_partials ? c->d_parts[b] : nullptr, c->seg_ws,
                                  c->seg_ws_bytes, c->compute);
    if (st != EXSUM_OK) break;
    if (cudaMemcpyAsync(c->h_out[b], c->d_out[b], ns * 8, cudaMemcpyDeviceToHost, c->compute) !=
            cudaSuccess ||
        (h_partials &&
         cudaMemcpyAsync(c->h_parts[b], c->d_parts[b], ns * sizeof(exsum_partial),
                         cudaMemcpyDeviceToHost, c->compute) != cudaSuccess) ||
        cudaEventRecord(c->consumed[b], c->compute) != cudaSuccess) {
      st = EXSUM_ECUDA;
      break;
    }
    pend0[b] = s0;
    pend1[b] = s1;
    pending[b] = true;
    for (size_t s = s0; s < s1; ++s)
      dev_terms += h_offsets[s + 1] > h_offsets[s] ? h_offsets[s + 1] - h_offsets[s] : 0;
  }
  for (int b = 0; b < kSlots; ++b)
    if (st == EXSUM_OK && !drain_slot(b)) st = EXSUM_ECUDA;
  if (cudaStreamSynchronize(c->compute) != cudaSuccess && st == EXSUM_OK) st = EXSUM_ECUDA;
  if (hybrid) c->pool->join_helpers();
  if (st != EXSUM_OK) {
    reset_after_error(c);
  } else {
    uint64_t total = 0;
    for (size_t s = 0; s < nseg; ++s)
      total += h_offsets[s + 1] > h_offsets[s] ? h_offsets[s + 1] - h_offsets[s] : 0;
    c->last_device_terms = dev_terms;
    c->last_host_terms = total - dev_terms;
  }
  cudaSetDevice(prev);
  return st;
}

int exsum_context_sum_file(exsum_context *c, const char *path, int format, double *h_result,
                           exsum_partial *h_partial, uint64_t *n_out) {
  EXSUM_NVTX("exsum_context_sum_file");
  if (!c || !path || (!h_result && !h_partial)) return EXSUM_EINVAL;
  if (format == EXSUM_FORMAT_TEXT) {
    double *v = nullptr;
    size_t n = 0;
    int st = exsum_read_values(path, format, &v, &n);
    if (st == EXSUM_OK) st = exsum_context_sum(c, v, n, h_result, h_partial);
    exsum_free_values(v);
    if (st == EXSUM_OK && n_out) *n_out = n;
    return st;
  }
  if (format != EXSUM_FORMAT_BIN) return EXSUM_EINVAL;
  // bin: validate like read_values (io.cpp:94-99), then stream disk -> pinned
  // bounce -> device (the disk, not the cores, bounds this path: device only)
  double *probe = nullptr;
  size_t dummy = 0;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return exsum_read_values(path, format, &probe, &dummy);  // sets the message
  const off_t size = lseek(fd, 0, SEEK_END);
  if (size < 0 || size % 8 != 0) {
    close(fd);
    return exsum_read_values(path, format, &probe, &dummy);
  }
  std::lock_guard<std::mutex> lk(c->busy);
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(c->device) != cudaSuccess) {
    close(fd);
    return EXSUM_ECUDA;
  }
  int st = ensure_bounce(c);
  const size_t n = static_cast<size_t>(size) / 8;
  size_t off = 0;
  for (int i = 0; off < n && st == EXSUM_OK; ++i) {
    const size_t len = (n - off < c->stage_elems) ? n - off : c->stage_elems;
    const int b = i % kSlots;
    // the bounce buffer and stage slot are free once chunk i - kSlots was consumed
    if (i >= kSlots && cudaEventSynchronize(c->consumed[b]) != cudaSuccess) {
      st = EXSUM_ECUDA;
      break;
    }
    size_t got = 0;
    char *dst = reinterpret_cast<char *>(c->host[b]);
    while (got < len * 8) {
      const ssize_t r = pread(fd, dst + got, len * 8 - got, static_cast<off_t>(off * 8 + got));
      if (r <= 0) break;
      got += static_cast<size_t>(r);
    }
    if (got != len * 8) {
      st = EXSUM_EIO;
      break;
    }
    if (cudaMemcpyAsync(c->stage[b], c->host[b], len * sizeof(double), cudaMemcpyHostToDevice,
                        c->copy) != cudaSuccess ||
        cudaEventRecord(c->copied[b], c->copy) != cudaSuccess ||
        cudaStreamWaitEvent(c->compute, c->copied[b], 0) != cudaSuccess) {
      st = EXSUM_ECUDA;
      break;
    }
    st = exsum_cuda_accumulate(c->stage[b], len, off, c->ws, c->ws_bytes, c->compute);
    if (st == EXSUM_OK && cudaEventRecord(c->consumed[b], c->compute) != cudaSuccess)
      st = EXSUM_ECUDA;
    off += len;
  }
  close(fd);
  if (st == EXSUM_OK)
    st = exsum_cuda_finalize(c->d_result, c->d_partial, c->ws, c->ws_bytes, c->compute);
  if (st == EXSUM_OK &&
      cudaMemcpyAsync(c->h_partial, c->d_partial, sizeof(exsum_partial), cudaMemcpyDeviceToHost,
                      c->compute) != cudaSuccess)
    st = EXSUM_ECUDA;
  if (cudaStreamSynchronize(c->compute) != cudaSuccess && st == EXSUM_OK) st = EXSUM_ECUDA;
  if (cudaStreamSynchronize(c->copy) != cudaSuccess && st == EXSUM_OK) st = EXSUM_ECUDA;
  if (st != EXSUM_OK) {
    reset_after_error(c);  // EIO mid-file leaves chunks in the workspace otherwise
  } else {
    if (h_partial) *h_partial = *c->h_partial;
    if (h_result) exsum_partial_round(c->h_partial, h_result);
    c->last_device_terms = n;
    c->last_host_terms = 0;
    if (n_out) *n_out = n;
  }
  cudaSetDevice(prev);
  return st;
}

const char *exsum_version(void) { return "exsum_b200 0.2.0 sm_100a"; }

}  // extern "C"
