// FP64 FMA throughput and latency on the GPU (microbenchmark for the SG
// operator's roofline): independent DFMA chains per thread, swept over
// warps per SM and chains per warp; one dependent chain for latency.
//   nvcc -O3 -arch=sm_100a -o tools/bin/bench_fp64 tools/bench_fp64.cu && tools/bin/bench_fp64
#include <cstdio>

#include <cuda_runtime.h>

template <int CH>
__global__ void fma_chains(double* out, int iters, double a, double b) {
  double v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < CH; ++c) v[c] = fma(v[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CH>
static void run(int warps, int sms) {
  double* out;
  cudaMalloc(&out, 1 << 20);
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_chains<CH><<<sms, warps * 32>>>(out, 16, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  fma_chains<CH><<<sms, warps * 32>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fmas = double(sms) * warps * 32 * iters * 8.0 * CH;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double per_sm_clk = fmas / sms / (ms * 1e-3 * clk * 1e3);
  std::printf("warps/SM %2d chains %2d: %7.2f TFMA/s  %6.1f FMA/clk/SM  (%.3f ms)\n", warps, CH, fmas / (ms * 1e-3) / 1e12,
              per_sm_clk, ms);
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {1, 2, 4, 8, 16, 32}) {
    run<1>(w, sms);
    run<4>(w, sms);
    run<8>(w, sms);
  }
  return 0;
}
