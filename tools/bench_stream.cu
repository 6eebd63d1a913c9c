// Microbenchmark: HBM streaming throughput of (a) a per-CTA TMA bulk-copy ring
// (cp.async.bulk + mbarrier, consumer-released stages) and (b) plain 128-bit
// LDG streaming, as a function of CTAs, stages and chunk size.  Used to size
// the interior-sweep pipeline.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void ring_kernel(const double* __restrict__ src, long long n_chunks, int chunk_doubles, int S,
                            double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* stage = (double*)sm;
  unsigned long long* full = (unsigned long long*)(sm + (size_t)S * chunk_doubles * 8);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const unsigned bytes = chunk_doubles * 8;
  long long mine = 0, issued = 0;
  auto issue = [&](long long c) {
    const int st = issued % S;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(stage + (size_t)st * chunk_doubles)),
                 "l"(src + c * chunk_doubles), "r"(bytes), "r"(su32(&full[st])));
    ++issued;
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < S; ++i) {
      const long long c = blockIdx.x + (long long)i * gridDim.x;
      if (c < n_chunks) issue(c);
    }
  double acc = 0;
  long long consumed = 0;
  for (long long c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const int st = consumed % S;
    const unsigned par = (consumed / S) & 1;
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
        su32(&full[st])), "r"(par));
    const double2* b = (const double2*)(stage + (size_t)st * chunk_doubles);
    for (int i = threadIdx.x; i < chunk_doubles / 2; i += blockDim.x) acc += b[i].x + b[i].y;
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long cn = c + (long long)S * gridDim.x;
      if (cn < n_chunks) issue(cn);
    }
    ++consumed;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void ldg_kernel(const double2* __restrict__ src, long long n2, double* out) {
  double acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(src + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const long long n = 1LL << 30;  // 8 GB
  double *src, *out;
  cudaMalloc(&src, n * 8);
  cudaMalloc(&out, 8);
  cudaMemset(src, 0, n * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    ldg_kernel<<<148 * 8, 256>>>((const double2*)src, n / 2, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  printf("LDG.128 grid-stride: %.0f GB/s\n", n * 8 / ms / 1e6);
  struct Cfg { int ctas_per_sm, S, chunk; int threads; };
  Cfg cfgs[] = {{1, 5, 4096, 512}, {1, 6, 4096, 512}, {1, 5, 4096, 256}, {2, 3, 4096, 256},
                {2, 6, 2048, 256}, {1, 12, 2048, 512}, {4, 3, 2048, 128}, {1, 3, 8192, 512}};
  for (auto c : cfgs) {
    const size_t smem = (size_t)c.S * c.chunk * 8 + 128;
    cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long chunks = n / c.chunk;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      ring_kernel<<<148 * c.ctas_per_sm, c.threads, smem>>>(src, chunks, c.chunk, c.S, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    cudaError_t e = cudaGetLastError();
    printf("TMA ring ctas/SM=%d stages=%d chunk=%dKB threads=%d: %.0f GB/s %s\n", c.ctas_per_sm, c.S,
           c.chunk * 8 / 1024, c.threads, n * 8 / ms / 1e6, e ? cudaGetErrorString(e) : "");
  }
  // fewer SMs (128 CTAs, as the C2 sweep)
  {
    const int S = 5, chunk = 4096;
    const size_t smem = (size_t)S * chunk * 8 + 128;
    cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEventRecord(a);
    ring_kernel<<<128, 512, smem>>>(src, n / chunk, chunk, S, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("TMA ring 128 CTAs stages=5 chunk=32KB: %.0f GB/s\n", n * 8 / ms / 1e6);
  }
  return 0;
}
