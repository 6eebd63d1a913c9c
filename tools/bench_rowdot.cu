// Microbenchmark: TMA bulk-copy ring + warp-per-row dot-product consumers
// (the interior-sweep inner loop) on synthetic chunks of R rows x Lr doubles.
// Variants isolate the consumer cost: 0 = full row dot + warp reduction,
// 1 = loads only, 2 = dot without reduction, 3 = FMAs with a register vector.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int VARIANT>
__global__ void __launch_bounds__(544) rowdot_kernel(const double* __restrict__ src, long long n_chunks, int R,
                                                     int Lr, double* out) {
  constexpr int S = 5, STG = 4096;
  extern __shared__ __align__(128) unsigned char sm[];
  double* stage = (double*)sm;
  unsigned long long* full = (unsigned long long*)(sm + S * STG * 8);
  unsigned long long* empty = full + 8;
  double* vec = (double*)(empty + 8);
  double* res = vec + 1024;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 1024; i += blockDim.x) vec[i] = 1.0 + i * 1e-3;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared.b64 [%0], 16;" ::"r"(su32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const unsigned bytes = R * Lr * 8;
  if (warp == 16) {
    long long issued = 0;
    for (long long c = blockIdx.x; c < n_chunks; c += gridDim.x, ++issued) {
      const int st = issued % S;
      if (issued >= S)
        asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
            su32(&empty[st])), "r"((unsigned)(((issued / S) - 1) & 1)));
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(bytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(stage + (size_t)st * STG)),
                     "l"(src + (c % 4096) * STG), "r"(bytes), "r"(su32(&full[st])));
      }
      __syncwarp();
    }
    return;
  }
  long long consumed = 0;
  double keep = 0;
  double2 vr[10];
  for (int m = 0; m < 10; ++m) vr[m] = make_double2(vec[2 * lane + 64 * m], vec[2 * lane + 64 * m + 1]);
  for (long long c = blockIdx.x; c < n_chunks; c += gridDim.x, ++consumed) {
    const int st = consumed % S;
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
        su32(&full[st])), "r"((unsigned)((consumed / S) & 1)));
    const double* buf = stage + (size_t)st * STG;
    for (int r = warp; r < R; r += 16) {
      const double2* row = (const double2*)(buf + r * Lr);
      const double2* v2 = (const double2*)(vec + (r & 3) * 2);
      const int n2 = Lr >> 1;
      double d0 = 0, d1 = 0, d2 = 0, d3 = 0;
      if (VARIANT == 3) {
#pragma unroll
        for (int m = 0; m < 10; ++m) {
          const int q = lane + 32 * m;
          if (q < n2) {
            const double2 a = row[q];
            d0 += a.x * vr[m].x;
            d1 += a.y * vr[m].y;
          }
        }
      } else {
        int q = lane;
        for (; q + 32 < n2; q += 64) {
          const double2 a = row[q], b = v2[q], cc = row[q + 32], e = v2[q + 32];
          if (VARIANT == 1) {
            d0 += a.x;
            d1 += cc.x;
          } else {
            d0 += a.x * b.x;
            d1 += a.y * b.y;
            d2 += cc.x * e.x;
            d3 += cc.y * e.y;
          }
        }
        if (q < n2) {
          const double2 a = row[q], b = v2[q];
          d0 += a.x * b.x;
          d1 += a.y * b.y;
        }
      }
      double d = (d0 + d1) + (d2 + d3);
      if (VARIANT == 0 || VARIANT == 3) d = wsum(d);
      if (lane == 0) res[r] = d;
      keep += d;
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&empty[st])));
  }
  if (keep == 1234.5) out[0] = keep;
}

int main() {
  const long long n = 1LL << 30;
  double *src, *out;
  cudaMalloc(&src, 4096LL * 4096 * 8);
  cudaMalloc(&out, 8);
  cudaMemset(src, 0, 4096LL * 4096 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct C { int R, Lr; };
  C cs[] = {{12, 340}, {6, 620}, {64, 64}, {32, 128}};
  const size_t smem = 5 * 4096 * 8 + 256 + 2048 * 8;
  auto run = [&](auto kern, const char* name, C c) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long chunks = n / (c.R * c.Lr);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      kern<<<128, 544, smem>>>(src, chunks, c.R, c.Lr, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    cudaError_t e = cudaGetLastError();
    printf("%-28s R=%3d Lr=%4d : %6.0f GB/s (%.1f GB/s per CTA) %s\n", name, c.R, c.Lr,
           chunks * c.R * c.Lr * 8.0 / ms / 1e6, chunks * c.R * c.Lr * 8.0 / ms / 1e6 / 128, e ? cudaGetErrorString(e) : "");
  };
  for (auto c : cs) {
    run(rowdot_kernel<0>, "dot+reduce (sweep)", c);
    run(rowdot_kernel<1>, "loads only", c);
    run(rowdot_kernel<2>, "dot, no reduce", c);
    if (c.Lr <= 640) run(rowdot_kernel<3>, "register vector + reduce", c);
  }
  return 0;
}
