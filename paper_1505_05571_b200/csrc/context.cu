// context.cu — exact sum of a HOST array through the device path.
//
// exsum_context_sum is the drop-in for exact_sum(values, ExactMethod::large)
// (vector_ops.cpp:121-130) when the caller's values live in host memory, as
// they do for every reference caller.  The array is streamed through a
// two-buffer device staging ring: the copy stream moves chunk i+1 host->device
// while the compute stream accumulates chunk i (exsum_cuda_accumulate with the
// chunk's global base index, so Inf/NaN order is preserved); one finalize
// launch rounds, and the 8-byte result (and optionally the 592-byte partial
// record) is copied back.  Pinned host memory gives full PCIe/C2C bandwidth;
// pageable memory works but is staged by the driver.

#include <cuda_runtime.h>
#include <fcntl.h>
#include <stdint.h>
#include <string.h>
#include <unistd.h>

#include <new>
#include <string>

#include "exsum_b200.h"

struct exsum_context {
  int device = 0;
  void *ws = nullptr;
  size_t ws_bytes = 0;
  double *stage[2] = {nullptr, nullptr};
  size_t stage_elems = 0;
  cudaStream_t copy = nullptr, compute = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
  double *d_result = nullptr;
  exsum_partial *d_partial = nullptr;
  double *host[2] = {nullptr, nullptr};  // pinned file-read buffers (first file sum)
  cudaEvent_t h2d[2] = {nullptr, nullptr};
};

namespace {

void destroy(exsum_context *c) {
  if (!c) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  for (int i = 0; i < 2; ++i) {
    if (c->host[i]) cudaFreeHost(c->host[i]);
    if (c->h2d[i]) cudaEventDestroy(c->h2d[i]);
    if (c->stage[i]) cudaFree(c->stage[i]);
    if (c->copied[i]) cudaEventDestroy(c->copied[i]);
    if (c->consumed[i]) cudaEventDestroy(c->consumed[i]);
  }
  if (c->ws) cudaFree(c->ws);
  if (c->d_result) cudaFree(c->d_result);
  if (c->d_partial) cudaFree(c->d_partial);
  if (c->copy) cudaStreamDestroy(c->copy);
  if (c->compute) cudaStreamDestroy(c->compute);
  cudaSetDevice(prev);
  delete c;
}

}  // namespace

extern "C" {

exsum_context *exsum_context_create(int device, size_t staging_bytes) {
  if (staging_bytes < (size_t{1} << 20)) staging_bytes = size_t{1} << 20;
  exsum_context *c = new (std::nothrow) exsum_context;
  if (!c) return nullptr;
  c->device = device;
  int prev = 0;
  cudaGetDevice(&prev);
  bool ok = cudaSetDevice(device) == cudaSuccess;
  c->stage_elems = staging_bytes / 2 / sizeof(double);
  c->stage_elems &= ~size_t{3};
  c->ws_bytes = exsum_cuda_workspace_bytes();
  ok = ok && cudaMalloc(&c->ws, c->ws_bytes) == cudaSuccess;
  ok = ok && cudaMalloc(&c->d_result, sizeof(double)) == cudaSuccess;
  ok = ok && cudaMalloc(&c->d_partial, sizeof(exsum_partial)) == cudaSuccess;
  for (int i = 0; i < 2 && ok; ++i) {
    ok = cudaMalloc(&c->stage[i], c->stage_elems * sizeof(double)) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->copied[i], cudaEventDisableTiming) == cudaSuccess;
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

int exsum_context_sum(exsum_context *c, const double *h_x, size_t n, double *h_result,
                      exsum_partial *h_partial) {
  return exsum_context_sum_at(c, h_x, n, 0, h_result, h_partial);
}

int exsum_context_sum_at(exsum_context *c, const double *h_x, size_t n, uint64_t base_index,
                         double *h_result, exsum_partial *h_partial) {
  if (!c || (n && !h_x) || (!h_result && !h_partial)) return EXSUM_EINVAL;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(c->device) != cudaSuccess) return EXSUM_ECUDA;
  int st = EXSUM_OK;
  size_t off = 0;
  int i = 0;
  while (off < n && st == EXSUM_OK) {
    const size_t len = (n - off < c->stage_elems) ? n - off : c->stage_elems;
    const int b = i & 1;
    if (cudaStreamWaitEvent(c->copy, c->consumed[b], 0) != cudaSuccess ||
        cudaMemcpyAsync(c->stage[b], h_x + off, len * sizeof(double), cudaMemcpyHostToDevice,
                        c->copy) != cudaSuccess ||
        cudaEventRecord(c->copied[b], c->copy) != cudaSuccess ||
        cudaStreamWaitEvent(c->compute, c->copied[b], 0) != cudaSuccess) {
      st = EXSUM_ECUDA;
      break;
    }
    st = exsum_cuda_accumulate(c->stage[b], len, base_index + off, c->ws, c->ws_bytes,
                               c->compute);
    if (st == EXSUM_OK && cudaEventRecord(c->consumed[b], c->compute) != cudaSuccess)
      st = EXSUM_ECUDA;
    off += len;
    ++i;
  }
  if (st == EXSUM_OK)
    st = exsum_cuda_finalize(c->d_result, c->d_partial, c->ws, c->ws_bytes, c->compute);
  if (st == EXSUM_OK && h_result &&
      cudaMemcpyAsync(h_result, c->d_result, sizeof(double), cudaMemcpyDeviceToHost,
                      c->compute) != cudaSuccess)
    st = EXSUM_ECUDA;
  if (st == EXSUM_OK && h_partial &&
      cudaMemcpyAsync(h_partial, c->d_partial, sizeof(exsum_partial), cudaMemcpyDeviceToHost,
                      c->compute) != cudaSuccess)
    st = EXSUM_ECUDA;
  if (cudaStreamSynchronize(c->compute) != cudaSuccess) st = EXSUM_ECUDA;
  cudaSetDevice(prev);
  return st;
}

int exsum_context_sum_file(exsum_context *c, const char *path, int format, double *h_result,
                           exsum_partial *h_partial, uint64_t *n_out) {
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
  // bin: validate like read_values (io.cpp:94-99), then stream
  double *probe = nullptr;
  size_t dummy = 0;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return exsum_read_values(path, format, &probe, &dummy);  // sets the message
  const off_t size = lseek(fd, 0, SEEK_END);
  if (size < 0 || size % 8 != 0) {
    close(fd);
    return exsum_read_values(path, format, &probe, &dummy);
  }
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(c->device) != cudaSuccess) {
    close(fd);
    return EXSUM_ECUDA;
  }
  int st = EXSUM_OK;
  for (int i = 0; i < 2 && st == EXSUM_OK; ++i) {
    if (!c->host[i] &&
        (cudaMallocHost(&c->host[i], c->stage_elems * sizeof(double)) != cudaSuccess ||
         cudaEventCreateWithFlags(&c->h2d[i], cudaEventDisableTiming) != cudaSuccess))
      st = EXSUM_ECUDA;
  }
  const size_t n = static_cast<size_t>(size) / 8;
  size_t off = 0;
  int i = 0;
  while (off < n && st == EXSUM_OK) {
    const size_t len = (n - off < c->stage_elems) ? n - off : c->stage_elems;
    const int b = i & 1;
    // the host buffer is free once its previous host->device copy completed
    if (i >= 2 && cudaEventSynchronize(c->h2d[b]) != cudaSuccess) {
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
    if (cudaStreamWaitEvent(c->copy, c->consumed[b], 0) != cudaSuccess ||
        cudaMemcpyAsync(c->stage[b], c->host[b], len * sizeof(double), cudaMemcpyHostToDevice,
                        c->copy) != cudaSuccess ||
        cudaEventRecord(c->h2d[b], c->copy) != cudaSuccess ||
        cudaEventRecord(c->copied[b], c->copy) != cudaSuccess ||
        cudaStreamWaitEvent(c->compute, c->copied[b], 0) != cudaSuccess) {
      st = EXSUM_ECUDA;
      break;
    }
    st = exsum_cuda_accumulate(c->stage[b], len, off, c->ws, c->ws_bytes, c->compute);
    if (st == EXSUM_OK && cudaEventRecord(c->consumed[b], c->compute) != cudaSuccess)
      st = EXSUM_ECUDA;
    off += len;
    ++i;
  }
  close(fd);
  if (st == EXSUM_OK)
    st = exsum_cuda_finalize(c->d_result, c->d_partial, c->ws, c->ws_bytes, c->compute);
  if (st == EXSUM_OK && h_result &&
      cudaMemcpyAsync(h_result, c->d_result, sizeof(double), cudaMemcpyDeviceToHost,
                      c->compute) != cudaSuccess)
    st = EXSUM_ECUDA;
  if (st == EXSUM_OK && h_partial &&
      cudaMemcpyAsync(h_partial, c->d_partial, sizeof(exsum_partial), cudaMemcpyDeviceToHost,
                      c->compute) != cudaSuccess)
    st = EXSUM_ECUDA;
  if (cudaStreamSynchronize(c->compute) != cudaSuccess && st == EXSUM_OK) st = EXSUM_ECUDA;
  if (cudaStreamSynchronize(c->copy) != cudaSuccess && st == EXSUM_OK) st = EXSUM_ECUDA;
  cudaSetDevice(prev);
  if (st == EXSUM_OK && n_out) *n_out = n;
  return st;
}

const char *exsum_version(void) { return "exsum_b200 0.1.0 sm_100a"; }

}  // extern "C"
