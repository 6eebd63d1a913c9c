// Cost of a kernel boundary for the phase-split PCG: back-to-back launches of
// a trivial kernel (one grid barrier) with the phase kernels' shape (2 CTAs
// per SM x 256 threads, ~100 KB dynamic shared memory each), cooperative vs
// plain, stream vs CUDA graph.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void coop_kernel(double* out, int zero_smem) {
  extern __shared__ double sm[];
  if (zero_smem)
    for (int i = threadIdx.x; i < zero_smem; i += blockDim.x) sm[i] = 0.0;
  cg::this_grid().sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] += sm[0];
}
__global__ void plain_kernel(double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] += 1.0;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  const int grid = 296, smem = 100 * 1024, reps = 200;
  cudaFuncSetAttribute((const void*)coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  for (int zero : {0, smem / 8}) {
    void* args[] = {&out, &zero};
    auto launch = [&]() { cudaLaunchCooperativeKernel((const void*)coop_kernel, grid, 256, args, smem, st); };
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(a, st);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cooperative, stream, zero_smem=%d: %.2f us per launch\n", zero, ms * 1e3 / reps);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < reps; ++i) launch();
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(a, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("cooperative, graph,  zero_smem=%d: %.2f us per launch\n", zero, ms * 1e3 / reps);
  }
  for (int i = 0; i < 10; ++i) plain_kernel<<<grid, 256, 0, st>>>(out);
  cudaEventRecord(a, st);
  for (int i = 0; i < reps; ++i) plain_kernel<<<grid, 256, 0, st>>>(out);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("plain, stream: %.2f us per launch\n", ms * 1e3 / reps);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
