// Allocation-cost probe: cudaMalloc / cudaMallocAsync / VMM map of large buffers.
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
static double ms(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
int main() {
  cudaFree(0);
  size_t fr, tot;
  cudaMemGetInfo(&fr, &tot);
  std::printf("free %.1f GB of %.1f\n", fr / 1e9, tot / 1e9);
  const size_t GB = 1ull << 30;
  for (int rep = 0; rep < 2; ++rep) {
    void* p;
    auto t0 = std::chrono::steady_clock::now();
    cudaMalloc(&p, 64 * GB);
    double a = ms(t0);
    t0 = std::chrono::steady_clock::now();
    cudaMemset(p, 0, 64 * GB);
    cudaDeviceSynchronize();
    double b = ms(t0);
    t0 = std::chrono::steady_clock::now();
    cudaFree(p);
    double c = ms(t0);
    std::printf("cudaMalloc 64GB %.1f ms, memset %.1f ms, free %.1f ms\n", a, b, c);
  }
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int rep = 0; rep < 3; ++rep) {
    void* p;
    auto t0 = std::chrono::steady_clock::now();
    cudaMallocAsync(&p, 64 * GB, s);
    cudaStreamSynchronize(s);
    double a = ms(t0);
    t0 = std::chrono::steady_clock::now();
    cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
    std::printf("cudaMallocAsync 64GB %.1f ms, free %.1f ms\n", a, ms(t0));
  }
  // 16 x 4 GB chunks
  {
    void* ps[16];
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 16; ++i) cudaMalloc(&ps[i], 4 * GB);
    std::printf("16 x cudaMalloc 4GB %.1f ms\n", ms(t0));
    for (int i = 0; i < 16; ++i) cudaFree(ps[i]);
  }
  return 0;
}
