// Sharded interface algebra: the point-to-point halo that
// completes a rank's partial interface sums (the reference's serial scatters
// src/dd.cpp:151-155, :222-226, :247-251, src/sg.cpp:306-311 become a local
// partial + an exchange with the neighbouring ranks), and the ownership mask
// of the interface dots (every global node counted once).
#include <algorithm>

#include "solver.cuh"
#include "tiles.cuh"

namespace sgw {

// pack every shared node's partial (all terms) into the peers' send blocks
__global__ void halo_pack_kernel(HaloDev H, const double* __restrict__ y, int nt) {
  const long long total = (long long)H.n_shared * nt;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int c = int(t % H.n_shared), j = int(t / H.n_shared);
    const int q = H.cnode[c];
    halo_pack_one(H, j, q, y[(long long)j * H.nloc + q]);
  }
}

__global__ void halo_combine_kernel(HaloDev H, double* __restrict__ y, int nt) {
  const long long total = (long long)H.n_shared * nt;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int c = int(t % H.n_shared), j = int(t / H.n_shared);
    double* yq = y + (long long)j * H.nloc + H.cnode[c];
    *yq = halo_combine_one(H, c, j, *yq);
  }
}

void GpuSolver::build_halo() {
  const Halo& h = G.halo;
  const int np = int(h.peers.size());
  hx_off_.assign(np, 0), hx_cnt_.assign(np, 0);
  std::vector<int> base(np);
  size_t tot = 0;
  for (int i = 0; i < np; ++i) {
    const int cnt = h.peer_off[i + 1] - h.peer_off[i];
    base[i] = int(tot);
    hx_off_[i] = tot, hx_cnt_[i] = size_t(cnt) * NT;
    tot += size_t(cnt) * NT;
  }
  // pack entries per local node (<= 3 peers share a node)
  std::vector<std::vector<int2>> per(G.n_iface);
  for (int i = 0; i < np; ++i) {
    const int cnt = h.peer_off[i + 1] - h.peer_off[i];
    for (int k = 0; k < cnt; ++k) per[h.idx[h.peer_off[i] + k]].push_back(make_int2(base[i] + k, cnt));
  }
  std::vector<int> pptr(G.n_iface + 1, 0);
  std::vector<int2> pk;
  for (int q = 0; q < G.n_iface; ++q) {
    pk.insert(pk.end(), per[q].begin(), per[q].end());
    pptr[q + 1] = int(pk.size());
  }
  std::vector<int2> cs;
  for (size_t e = 0; e < h.src_rank.size(); ++e) {
    if (h.src_pos[e] < 0) {
      cs.push_back(make_int2(-1, 0));
      continue;
    }
    const int i = int(std::find(h.peers.begin(), h.peers.end(), h.src_rank[e]) - h.peers.begin());
    const int cnt = h.peer_off[i + 1] - h.peer_off[i];
    cs.push_back(make_int2(base[i] + h.src_pos[e], cnt));
  }
  hx_pk_ptr_.upload(pptr), hx_pk_.upload(pk.empty() ? std::vector<int2>{make_int2(0, 0)} : pk);
  hx_cnode_.upload(h.node.empty() ? std::vector<int>{0} : h.node);
  hx_cptr_.upload(h.src_ptr);
  hx_csrc_.upload(cs.empty() ? std::vector<int2>{make_int2(-1, 0)} : cs);
  hx_send_.alloc(std::max<size_t>(1, tot)), hx_recv_.alloc(std::max<size_t>(1, tot));
  hx_send_.zero(st_), hx_recv_.zero(st_);
  hx_nshared_ = int(h.node.size());
  iface_gpos_d_.upload(G.iface_gpos);
  // dots over the interface: each global node once (its lowest-rank holder)
  if (comm_) {
    std::vector<double> w((size_t)NG);
    for (int j = 0; j < NT; ++j)
      for (int q = 0; q < G.n_iface; ++q) w[(size_t)j * G.n_iface + q] = G.iface_owner[q] == G.rank ? 1.0 : 0.0;
    own_w_.upload(w);
  }
}

HaloDev GpuSolver::halo_dev() const {
  return HaloDev{G.n_iface, hx_nshared_, hx_pk_ptr_.p, hx_pk_.p, hx_cnode_.p, hx_cptr_.p, hx_csrc_.p, hx_send_.p,
                 hx_recv_.p};
}

void GpuSolver::halo_exchange() {
  comm_->exchange(G.halo.peers, hx_off_, hx_cnt_, hx_send_.p, hx_recv_.p, st_);
}

// y (local partial interface vector over this rank's subdomains) -> the full
// sums on every node this rank holds
void GpuSolver::halo_sum(double* y) {
  if (!comm_ || G.halo.peers.empty()) return;
  const long long tot = (long long)hx_nshared_ * NT;
  const int grid = (int)std::min<long long>(std::max<long long>(1, (tot + 255) / 256), 4 * kNumSMs);
  halo_pack_kernel<<<grid, 256, 0, st_>>>(halo_dev(), y, NT);
  SGW_LAUNCHED();
  halo_exchange();
  halo_combine_kernel<<<grid, 256, 0, st_>>>(halo_dev(), y, NT);
  SGW_LAUNCHED();
}

// global interface vector (term-major over all n_iface_global nodes) -> this
// rank's local numbering, and back (owned entries + a sum over ranks, so every
// rank returns the whole vector)
__global__ void iface_to_local_kernel(const double* __restrict__ g, double* __restrict__ l, const int* __restrict__ gpos,
                                      int nloc, int nglob, long long NG) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NG; t += (long long)gridDim.x * blockDim.x) {
    const long long j = t / nloc;
    l[t] = g[j * nglob + gpos[t % nloc]];
  }
}
__global__ void iface_to_global_kernel(const double* __restrict__ l, double* __restrict__ g, const int* __restrict__ gpos,
                                       const double* __restrict__ own, int nloc, int nglob, long long NG) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NG; t += (long long)gridDim.x * blockDim.x) {
    const long long j = t / nloc;
    if (!own || own[t] != 0.0) g[j * nglob + gpos[t % nloc]] = l[t];
  }
}

void GpuSolver::iface_to_local(const double* glob, double* loc) {
  if (!comm_) {
    SGW_CUDA(cudaMemcpyAsync(loc, glob, NG * sizeof(double), cudaMemcpyDeviceToDevice, st_));
    return;
  }
  iface_to_local_kernel<<<std::max(1, std::min(cdiv(NG, 256), 4096)), 256, 0, st_>>>(glob, loc, iface_gpos_d_.p,
                                                                                   G.n_iface, G.n_iface_global, NG);
  SGW_LAUNCHED();
}

void GpuSolver::iface_to_global(const double* loc, double* glob) {
  if (!comm_) {
    SGW_CUDA(cudaMemcpyAsync(glob, loc, NG * sizeof(double), cudaMemcpyDeviceToDevice, st_));
    return;
  }
  SGW_CUDA(cudaMemsetAsync(glob, 0, NGG * sizeof(double), st_));
  iface_to_global_kernel<<<std::max(1, std::min(cdiv(NG, 256), 4096)), 256, 0, st_>>>(
      loc, glob, iface_gpos_d_.p, own_w_.p, G.n_iface, G.n_iface_global, NG);
  SGW_LAUNCHED();
  allreduce(glob, NGG);
}

}  // namespace sgw
