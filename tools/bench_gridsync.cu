// Cost of one cooperative-groups grid barrier on B200 at the persistent PCG's
// launch shape (2 CTAs x 256 threads per SM), vs a hand-rolled
// sense-reversing barrier (one red.release per CTA, acquire polling).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int n, double* sink) {
  cg::grid_group g = cg::this_grid();
  double v = threadIdx.x;
  for (int i = 0; i < n; ++i) {
    v += 1.0;
    g.sync();
  }
  if (v < 0) sink[0] = v;
}

__device__ unsigned g_count, g_gen;
__global__ void k_own(int n, double* sink) {
  double v = threadIdx.x;
  unsigned gen = 0;
  for (int i = 0; i < n; ++i) {
    v += 1.0;
    __syncthreads();
    if (threadIdx.x == 0) {
      gen = i + 1;
      unsigned arrived;
      asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(&g_count) : "memory");
      if (arrived == gridDim.x * gen - 1) {
        asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&g_gen), "r"(gen) : "memory");
      } else {
        unsigned cur;
        do {
          asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(&g_gen) : "memory");
        } while (cur < gen);
      }
    }
    __syncthreads();
  }
  if (v < 0) sink[0] = v;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  for (int bps : {1, 2}) {
    int grid = sms * bps, n = 2000;
    void* args[] = {&n, &sink};
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_cg, grid, 256, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      unsigned z = 0;
      cudaMemcpyToSymbol(g_count, &z, 4), cudaMemcpyToSymbol(g_gen, &z, 4);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_own, grid, 256, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms2;
      cudaEventElapsedTime(&ms2, a, b);
      if (rep) printf("grid %d CTAs x 256: cg::grid sync %.2f us, own barrier %.2f us (%s)\n", grid, ms * 1e3 / n,
                      ms2 * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
