// Sum-allreduce over the ranks that share one SG interface problem.
//
// The sharded solver (one GpuSolver per rank, each owning a contiguous range
// of subdomains) keeps every interface-space vector replicated.  The only
// exchange is the sum over subdomains that the reference performs in its
// scatters: R^T S R p (dd.cpp:151-155), B^T d (dd.cpp:221-226),
// sum R^T D zeta (dd.cpp:246-250), the step right-hand side (sg.cpp:306-311)
// and the one-off coarse matrix F_cc (dd.cpp:128-137).  Each of those becomes
// a local partial sum over owned subdomains followed by allreduce_sum.
//
//  * NcclComm: one process per GPU, ncclAllReduce on the solver's stream.
//  * ThreadComm: W solvers in one process on one device, each driven by its
//    own host thread; used to exercise the sharded path where only one GPU
//    exists.  The exchange is host-synchronised (no kernel waits on another
//    rank's kernel) and sums in ascending rank order.
#pragma once
#include <cuda_runtime.h>

#include <memory>

namespace sgw {

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t st) = 0;  // in place, device buffer
  virtual bool capturable() const = 0;  // may be recorded into a CUDA graph (stream-ordered, no host sync)
};

void nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(const void* id128, int rank, int world, int device);

struct ThreadGroup;
std::shared_ptr<ThreadGroup> make_thread_group(int world);
std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<ThreadGroup> group, int rank);

}  // namespace sgw
