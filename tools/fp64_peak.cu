// fp64_peak.cu -- FP64 roofline denominators for the FP64-bound paths (ACA build,
// matrix-free near field, DMMA multi-RHS), measured on the box:
//
//   dfma   : independent DFMA chains, 2 flop per thread-instruction
//   dadd   : independent DADD chains (the -fmad=false kernels are mostly DADD/DMUL)
//   dmul   : independent DMUL chains
//   dmma   : mma.sync.aligned.m8n8k4.row.col.f64 back to back (2*8*8*4 flop per warp-MMA)
//   lat    : one dependent DFMA chain per warp (latency in cycles per DFMA)
//   div    : __ddiv_rn throughput (thread-divisions/s), the K1 series' per-term division
//
// Prints one JSON line.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(256) thr_kernel(double* out, double seed) {
  double a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = seed + threadIdx.x * 1e-9 + c * 1e-7;
  const double b = 0.999999999, cc = 1e-12;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if constexpr (OP == 0) a[c] = __fma_rn(a[c], b, cc);
      else if constexpr (OP == 1) a[c] = __dadd_rn(a[c], cc);
      else a[c] = __dmul_rn(a[c], b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += a[c];
  if (s == 12345.0) out[0] = s;
}

__global__ void __launch_bounds__(256) div_kernel(double* out, double seed) {
  double a[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) a[c] = seed + threadIdx.x * 1e-9 + c * 1e-7;
  const double b = 1.0000001;
  for (int it = 0; it < kIters / 8; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = __ddiv_rn(a[c], b);
  }
  double s = a[0] + a[1] + a[2] + a[3];
  if (s == 12345.0) out[0] = s;
}

__global__ void lat_kernel(double* out, double seed, long long* cycles) {
  double a = seed + threadIdx.x;
  const double b = 0.999999999, c = 1e-12;
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) a = __fma_rn(a, b, c);
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
  if (a == 12345.0) out[0] = a;
}

__global__ void __launch_bounds__(256) dmma_kernel(double* out, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double acc[4][2] = {};
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 4; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  double* out;
  long long* cyc;
  CK(cudaMalloc(&out, 64));
  CK(cudaMalloc(&cyc, 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256;
  auto timeit = [&](auto launch) -> double {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return best * 1e-3;
  };
  const double thr_ops = static_cast<double>(blocks) * threads * kChains * kIters;
  const double t_fma = timeit([&] { thr_kernel<0><<<blocks, threads>>>(out, 1.0); });
  const double t_add = timeit([&] { thr_kernel<1><<<blocks, threads>>>(out, 1.0); });
  const double t_mul = timeit([&] { thr_kernel<2><<<blocks, threads>>>(out, 1.0); });
  const double t_div = timeit([&] { div_kernel<<<blocks, threads>>>(out, 1.0); });
  const double t_mma = timeit([&] { dmma_kernel<<<blocks, threads>>>(out, 1.0); });
  lat_kernel<<<1, 32>>>(out, 1.0, cyc);
  CK(cudaDeviceSynchronize());
  long long cycles = 0;
  CK(cudaMemcpy(&cycles, cyc, 8, cudaMemcpyDeviceToHost));
  const double warps_mma = static_cast<double>(blocks) * (threads / 32) * 4 * kIters;
  const double div_ops = static_cast<double>(blocks) * threads * 4 * (kIters / 8);
  std::printf(
      "{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"dfma_tflops\": %.3f, \"dfma_inst_per_s\": %.4e, "
      "\"dadd_inst_per_s\": %.4e, \"dmul_inst_per_s\": %.4e, \"fp64_inst_per_clk_per_sm_at_attr_clock\": %.2f, "
      "\"ddiv_rn_per_s\": %.4e, \"dmma_tflops\": %.3f, \"dfma_dep_latency_cycles\": %.2f}\n",
      sms, clk_khz / 1e3, 2.0 * thr_ops / t_fma / 1e12, thr_ops / t_fma, thr_ops / t_add, thr_ops / t_mul,
      thr_ops / t_fma / (sms * clk_khz * 1e3), div_ops / t_div, warps_mma * 2.0 * 8 * 8 * 4 / t_mma / 1e12,
      static_cast<double>(cycles) / kIters);
  return 0;
}
