// Exchanges between the ranks that share one SG interface problem.
//
// The sharded solver (one GpuSolver per rank, each owning a 2D block of
// subdomains, host.hpp Geometry) holds the interface nodes its subdomains
// touch.  The reference's subdomain sums become:
//  * interface sums R^T S R p (dd.cpp:151-155), sum R^T D zeta (dd.cpp:246-250)
//    and the step right-hand side (sg.cpp:306-311): a local partial over owned
//    subdomains, then a point-to-point halo exchange of the partials of the
//    nodes shared with neighbouring ranks (exchange());
//  * the coarse vector B^T d (dd.cpp:221-226), the CG scalars and once the
//    coarse matrix F_cc (dd.cpp:128-137): allreduce_sum.
//
//  * NcclComm: one process per GPU; grouped ncclSend/ncclRecv and
//    ncclAllReduce on the solver's stream (graph-capturable).
//  * ThreadComm: W solvers in one process on one device, each driven by its
//    own host thread; used to exercise the sharded path where only one GPU
//    exists.  Host-synchronised (no kernel waits on another rank's kernel).
//  * SoloComm: one rank of a W-rank decomposition constructed alone (no
//    peers present): exchanges deliver zeros.  Construction / memory and
//    kernel timing of a shard only; the results are not physical.
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <vector>

namespace sgw {

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t st) = 0;  // in place, device buffer
  virtual bool capturable() const = 0;  // may be recorded into a CUDA graph (stream-ordered, no host sync)
  // point-to-point: for each i, send send[off[i] .. off[i]+cnt[i]) to peers[i]
  // and receive the same-sized block from it into recv[off[i] ..)
  virtual void exchange(const std::vector<int>& peers, const std::vector<size_t>& off,
                        const std::vector<size_t>& cnt, const double* send, double* recv, cudaStream_t st) = 0;
  // raise Error(ENCCL) if the transport failed asynchronously (and abort it)
  virtual void poll() {}
  virtual bool solo() const { return false; }
};

void nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(const void* id128, int rank, int world, int device);

struct ThreadGroup;
std::shared_ptr<ThreadGroup> make_thread_group(int world);
void thread_group_abort(ThreadGroup& g);  // a failed rank releases the others (their collectives throw)
std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<ThreadGroup> group, int rank);
std::unique_ptr<Comm> make_solo_comm(int rank, int world);

}  // namespace sgw
