// Shared helpers for the sm_100a SG-PCG kernels.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges show up under Nsight Systems / Compute, no-ops otherwise

namespace sgw {

// NVTX range over a host scope (setup phases, the phases of a Newmark step).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Status-carrying exception; capi.cpp maps it to the sgw_status codes.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SGW_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::sgw::Error(4, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                                __FILE__ + ":" + std::to_string(__LINE__));              \
  } while (0)

// Every kernel launch of the library goes through this counter so that the
// benchmark can report how many of our kernels ran in a timed region.
extern std::atomic<long long> g_launches;
#define SGW_LAUNCHED()                \
  do {                                \
    ++::sgw::g_launches;              \
    SGW_CUDA(cudaPeekAtLastError());  \
  } while (0)

constexpr int kNumSMs = 148;
constexpr int kTile = 64;  // tile edge of the packed symmetric matrices

inline int cdiv(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-function, process-wide
// setting: solvers of one process (e.g. LocalGroup ranks with different local
// sizes) must leave it at the largest size any of them launches with.
inline void ensure_dyn_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<const void*, size_t> cur;
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[fn];
  if (bytes > c) {
    SGW_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    c = bytes;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace sgw
