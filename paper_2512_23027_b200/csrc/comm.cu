// Comm implementations (see comm.hpp).
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.hpp"
#include "common.cuh"

namespace sgw {

#define SGW_NCCL(call)                                                                                      \
  do {                                                                                                      \
    ncclResult_t r_ = (call);                                                                               \
    if (r_ != ncclSuccess) throw Error(5, std::string("NCCL: ") + ncclGetErrorString(r_) + " at " + __FILE__ + \
                                              ":" + std::to_string(__LINE__));                              \
  } while (0)

void nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  SGW_NCCL(ncclGetUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
}

namespace {
class NcclComm final : public Comm {
 public:
  NcclComm(const void* id128, int rank, int world, int device) : rank_(rank), world_(world) {
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    SGW_CUDA(cudaSetDevice(device));
    SGW_NCCL(ncclCommInitRank(&comm_, world, id, rank));
  }
  ~NcclComm() override {
    if (comm_) ncclCommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int size() const override { return world_; }
  bool capturable() const override { return true; }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    if (n == 0) return;
    SGW_NCCL(ncclAllReduce(buf, buf, n, ncclDouble, ncclSum, comm_, st));
  }

 private:
  ncclComm_t comm_ = nullptr;
  int rank_, world_;
};

__global__ void sum_ranks_kernel(const double* const* __restrict__ src, int world, size_t n, double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r < world; ++r) acc += src[r][i];  // ascending rank order
    out[i] = acc;
  }
}
}  // namespace

struct ThreadGroup {
  explicit ThreadGroup(int w) : world(w), slot(w, nullptr) {}
  int world;
  std::vector<double*> slot;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

std::shared_ptr<ThreadGroup> make_thread_group(int world) { return std::make_shared<ThreadGroup>(world); }

namespace {
class ThreadComm final : public Comm {
 public:
  ThreadComm(std::shared_ptr<ThreadGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}
  ~ThreadComm() override {
    if (tmp_) cudaFree(tmp_);
    if (ptrs_) cudaFree(ptrs_);
  }
  int rank() const override { return rank_; }
  int size() const override { return g_->world; }
  bool capturable() const override { return false; }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    if (n == 0) return;
    if (n > cap_) {
      if (tmp_) cudaFree(tmp_);
      SGW_CUDA(cudaMalloc(&tmp_, n * sizeof(double)));
      cap_ = n;
    }
    if (!ptrs_) SGW_CUDA(cudaMalloc(&ptrs_, g_->world * sizeof(double*)));
    SGW_CUDA(cudaStreamSynchronize(st));  // this rank's partial is final
    g_->slot[rank_] = buf;
    g_->barrier();  // every rank's partial is final
    SGW_CUDA(cudaMemcpyAsync(ptrs_, g_->slot.data(), g_->world * sizeof(double*), cudaMemcpyHostToDevice, st));
    sum_ranks_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 1184), 256, 0, st>>>(ptrs_, g_->world, n, tmp_);
    SGW_LAUNCHED();
    SGW_CUDA(cudaStreamSynchronize(st));
    g_->barrier();  // nobody overwrites its partial while another rank still reads it
    SGW_CUDA(cudaMemcpyAsync(buf, tmp_, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }

 private:
  std::shared_ptr<ThreadGroup> g_;
  int rank_;
  double* tmp_ = nullptr;
  double** ptrs_ = nullptr;
  size_t cap_ = 0;
};
}  // namespace

std::unique_ptr<Comm> make_nccl_comm(const void* id128, int rank, int world, int device) {
  return std::make_unique<NcclComm>(id128, rank, world, device);
}
std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<ThreadGroup> group, int rank) {
  return std::make_unique<ThreadComm>(std::move(group), rank);
}

}  // namespace sgw
