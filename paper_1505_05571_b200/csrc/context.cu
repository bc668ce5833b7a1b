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
#include <stdint.h>
#include <string.h>

#include <new>

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
};

namespace {

void destroy(exsum_context *c) {
  if (!c) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  for (int i = 0; i < 2; ++i) {
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
    st = exsum_cuda_accumulate(c->stage[b], len, off, c->ws, c->ws_bytes, c->compute);
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

const char *exsum_version(void) { return "exsum_b200 0.1.0 sm_100a"; }

}  // extern "C"
