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
    if (n == 0 || world_ == 1) return;  // a sum over one rank is the identity
    SGW_NCCL(ncclAllReduce(buf, buf, n, ncclDouble, ncclSum, comm_, st));
  }
  void exchange(const std::vector<int>& peers, const std::vector<size_t>& off, const std::vector<size_t>& cnt,
                const double* send, double* recv, cudaStream_t st) override {
    if (peers.empty()) return;
    SGW_NCCL(ncclGroupStart());
    for (size_t i = 0; i < peers.size(); ++i) {
      SGW_NCCL(ncclSend(send + off[i], cnt[i], ncclDouble, peers[i], comm_, st));
      SGW_NCCL(ncclRecv(recv + off[i], cnt[i], ncclDouble, peers[i], comm_, st));
    }
    SGW_NCCL(ncclGroupEnd());
  }
  // ncclCommGetAsyncError: a peer that died or a failed transfer surfaces
  // here; abort the communicator so no later call blocks on it
  void poll() override {
    if (!comm_) throw Error(5, "NCCL communicator was aborted");
    ncclResult_t async = ncclSuccess;
    SGW_NCCL(ncclCommGetAsyncError(comm_, &async));
    if (async != ncclSuccess && async != ncclInProgress) {
      ncclCommAbort(comm_);
      comm_ = nullptr;
      throw Error(5, std::string("NCCL asynchronous error: ") + ncclGetErrorString(async));
    }
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
  explicit ThreadGroup(int w) : world(w), slot(w, nullptr), xsend(w, nullptr), xpeers(w), xoff(w) {}
  int world;
  std::vector<double*> slot;
  // exchange(): every rank's send buffer and its (peer, offset) blocks
  std::vector<const double*> xsend;
  std::vector<std::vector<int>> xpeers;
  std::vector<std::vector<size_t>> xoff;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  bool broken = false;  // a rank failed: every barrier throws from now on
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) throw Error(5, "local group aborted (another rank failed)");
    const long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen || broken; });
      if (generation == gen) throw Error(5, "local group aborted (another rank failed)");
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
};

void thread_group_abort(ThreadGroup& g) { g.abort(); }

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
  void exchange(const std::vector<int>& peers, const std::vector<size_t>& off, const std::vector<size_t>& cnt,
                const double* send, double* recv, cudaStream_t st) override {
    SGW_CUDA(cudaStreamSynchronize(st));  // this rank's send blocks are final
    g_->xsend[rank_] = send;
    g_->xpeers[rank_] = peers;
    g_->xoff[rank_] = off;
    g_->barrier();
    for (size_t i = 0; i < peers.size(); ++i) {  // the block peer i packed for this rank
      const int pr = peers[i];
      const auto& pp = g_->xpeers[pr];
      const size_t k = size_t(std::find(pp.begin(), pp.end(), rank_) - pp.begin());
      if (k == pp.size()) throw Error(1, "halo plan is not symmetric");
      SGW_CUDA(cudaMemcpyAsync(recv + off[i], g_->xsend[pr] + g_->xoff[pr][k], cnt[i] * sizeof(double),
                               cudaMemcpyDeviceToDevice, st));
    }
    SGW_CUDA(cudaStreamSynchronize(st));
    g_->barrier();  // nobody overwrites its send buffer while a peer still reads it
  }

 private:
  std::shared_ptr<ThreadGroup> g_;
  int rank_;
  double* tmp_ = nullptr;
  double** ptrs_ = nullptr;
  size_t cap_ = 0;
};
}  // namespace

namespace {
class SoloComm final : public Comm {
 public:
  SoloComm(int rank, int world) : rank_(rank), world_(world) {}
  int rank() const override { return rank_; }
  int size() const override { return world_; }
  bool capturable() const override { return true; }
  bool solo() const override { return true; }
  void allreduce_sum(double*, size_t, cudaStream_t) override {}
  void exchange(const std::vector<int>&, const std::vector<size_t>& off, const std::vector<size_t>& cnt, const double*,
                double* recv, cudaStream_t st) override {
    for (size_t i = 0; i < off.size(); ++i)
      if (cnt[i]) SGW_CUDA(cudaMemsetAsync(recv + off[i], 0, cnt[i] * sizeof(double), st));
  }

 private:
  int rank_, world_;
};
}  // namespace

std::unique_ptr<Comm> make_solo_comm(int rank, int world) { return std::make_unique<SoloComm>(rank, world); }

std::unique_ptr<Comm> make_nccl_comm(const void* id128, int rank, int world, int device) {
  return std::make_unique<NcclComm>(id128, rank, world, device);
}
std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<ThreadGroup> group, int rank) {
  return std::make_unique<ThreadComm>(std::move(group), rank);
}

}  // namespace sgw
