// host_mix.cu — host memory bandwidth probe for the hybrid host+device e2e design.
//
// Measures on the GPU box: (1) pinned host->device copy alone, (2) a T-thread
// streaming read (u64 sum) of a host array alone, for T in 1..nproc, (3) both at
// once (does the DMA share the host memory bandwidth with the CPU reads?),
// (4) pageable->device cudaMemcpy, (5) T-thread memcpy pageable->pinned.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fopenmp \
//        -o host_mix host_mix.cu && ./host_mix [GB]
#include <cuda_runtime.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

static uint64_t sink;

static double cpu_read(const uint64_t *x, size_t n, int T, int reps) {
  double t0 = now();
  uint64_t tot = 0;
  for (int r = 0; r < reps; ++r) {
#pragma omp parallel for num_threads(T) reduction(+ : tot) schedule(static)
    for (size_t i = 0; i < n; ++i) tot += x[i];
  }
  double el = now() - t0;
  sink += tot;
  return 8.0 * n * reps / el / 1e9;
}

int main(int argc, char **argv) {
  double gb = argc > 1 ? atof(argv[1]) : 4.0;
  size_t n = (size_t)(gb * 1e9 / 8);
  int nproc = omp_get_num_procs();
  printf("nproc %d, array %.2f GB\n", nproc, 8.0 * n / 1e9);
  uint64_t *h = nullptr, *pg = (uint64_t *)aligned_alloc(4096, n * 8);
  cudaMallocHost(&h, n * 8);
  void *d = nullptr;
  cudaMalloc(&d, n * 8);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) h[i] = pg[i] = i * 0x9E3779B97F4A7C15ull;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // (1) H2D alone
  for (int w = 0; w < 2; ++w) cudaMemcpyAsync(d, h, n * 8, cudaMemcpyHostToDevice, s);
  cudaEventRecord(a, s);
  for (int r = 0; r < 3; ++r) cudaMemcpyAsync(d, h, n * 8, cudaMemcpyHostToDevice, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double h2d = 3 * 8.0 * n / (ms / 1e3) / 1e9;
  printf("H2D pinned alone: %.1f GB/s\n", h2d);
  // (2) CPU read alone
  for (int T = 1; T <= nproc; T *= 2) printf("cpu read T=%d: %.1f GB/s\n", T, cpu_read(pg, n, T, 3));
  if ((nproc & (nproc - 1)) != 0) printf("cpu read T=%d: %.1f GB/s\n", nproc, cpu_read(pg, n, nproc, 3));
  printf("cpu read pinned T=%d: %.1f GB/s\n", nproc, cpu_read(h, n, nproc, 3));
  // (3) both: H2D loop in a thread while the CPU reads T-1 / T threads
  for (int T : {nproc - 1, nproc}) {
    std::atomic<bool> stop{false};
    std::atomic<long> copies{0};
    std::thread dma([&] {
      while (!stop.load()) {
        cudaMemcpyAsync(d, h, n * 8 / 4, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        copies++;
      }
    });
    std::this_thread::sleep_for(std::chrono::milliseconds(50));
    long c0 = copies.load();
    double t0 = now();
    double cpu = cpu_read(pg, n, T, 4);
    double el = now() - t0;
    long c1 = copies.load();
    stop = true;
    dma.join();
    printf("concurrent: cpu T=%d %.1f GB/s + H2D %.1f GB/s\n", T, cpu,
           (c1 - c0) * 8.0 * n / 4 / el / 1e9);
  }
  // (4) pageable H2D
  cudaMemcpy(d, pg, n * 8, cudaMemcpyHostToDevice);
  double t0 = now();
  cudaMemcpy(d, pg, n * 8, cudaMemcpyHostToDevice);
  printf("H2D pageable cudaMemcpy: %.1f GB/s\n", 8.0 * n / (now() - t0) / 1e9);
  // (5) memcpy pageable -> pinned with T threads
  for (int T : {1, 4, 8, nproc}) {
    double t1 = now();
#pragma omp parallel num_threads(T)
    {
      int id = omp_get_thread_num(), nt = omp_get_num_threads();
      size_t b0 = n * id / nt, b1 = n * (id + 1) / nt;
      memcpy(h + b0, pg + b0, (b1 - b0) * 8);
    }
    printf("memcpy pageable->pinned T=%d: %.1f GB/s\n", T, 8.0 * n / (now() - t1) / 1e9);
  }
  // (6) cudaHostRegister cost
  t0 = now();
  cudaError_t e = cudaHostRegister(pg, n * 8, cudaHostRegisterDefault);
  double reg = now() - t0;
  t0 = now();
  cudaHostUnregister(pg);
  printf("cudaHostRegister %.2f GB: %.3f s (%s), unregister %.3f s\n", 8.0 * n / 1e9, reg,
         cudaGetErrorString(e), now() - t0);
  printf("sink %llu\n", (unsigned long long)(sink & 1));
  return 0;
}
