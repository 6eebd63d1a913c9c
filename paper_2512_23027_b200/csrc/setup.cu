// GPU setup of the SG interface system (src/sg.cpp:128-250, src/dd.cpp:98-140):
//  * block-tridiagonal Cholesky of every subdomain's flattened interior block
//    A_II (grid-row blocks B = W (P+1), node-major / term-minor),
//  * dense local Schur S_s = A_GG - (L^-1 A_IG)^T (L^-1 A_IG) by a rolling
//    block forward substitution (only two block rows of L^-1 A_IG live),
//  * NN2 data Q_s = S_rr^-1, Psi_s = Q_s S_rc, F_cc^-1,
//  * packing of S_s and Q_s into lower 64x64 tiles for the PCG SYMV.
// Dense factor/solve/GEMM steps are plain library calls (cuBLAS / cuSOLVER);
// assembly, extraction and packing are our kernels.  Not on the per-step path.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include <cstdio>

#include "solver.cuh"

namespace sgw {

void pack_tiles_range(TilePack& tp, int s, const double* src, int ld, cudaStream_t st);

#define SGW_BLAS(call)                                                                            \
  do {                                                                                            \
    cublasStatus_t s_ = (call);                                                                   \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                              \
      throw Error(4, "cuBLAS error " + std::to_string(int(s_)) + " at " + __FILE__ + ":" +          \
                         std::to_string(__LINE__));                                               \
  } while (0)
#define SGW_SOLVER(call)                                                                          \
  do {                                                                                            \
    cusolverStatus_t s_ = (call);                                                                 \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                            \
      throw Error(4, "cuSOLVER error " + std::to_string(int(s_)) + " at " + __FILE__ + ":" +        \
                         std::to_string(__LINE__));                                               \
  } while (0)

// Neighbour directions of the 7-point P1 pattern on a structured grid:
// 0 self, 1 E, 2 W, 3 N, 4 S, 5 NE, 6 SW.  Coefficients of the (symmetric)
// local operator are read from the node that owns the coupling.
__constant__ int kDI[7] = {0, 1, -1, 0, 0, 1, -1};
__constant__ int kDJ[7] = {0, 0, 0, 1, -1, 1, -1};

// Coupling coefficient of local stencil arrays (stride nl between components)
// from node lid towards direction dir; own = lid, nb = neighbour lid.
__device__ __forceinline__ double kcoef(const double* K, int nl, int lid, int nb, int dir) {
  switch (dir) {
    case 0: return K[lid];
    case 1: return K[nl + lid];
    case 2: return K[nl + nb];
    case 3: return K[2 * nl + lid];
    case 4: return K[2 * nl + nb];
    default: return 0.0;  // NE/SW stiffness couplings vanish on this mesh
  }
}
__device__ __forceinline__ double mcoef(const double* M, int nl, int lid, int nb, int dir) {
  switch (dir) {
    case 0: return M[lid];
    case 1: return M[nl + lid];
    case 2: return M[nl + nb];
    case 3: return M[2 * nl + lid];
    case 4: return M[2 * nl + nb];
    case 5: return M[3 * nl + lid];
    default: return M[3 * nl + nb];
  }
}

// Transient-operator block entry (row term kt, col term jt) between lid and nb:
// delta ms M + sum_i (ss g_i) K_i  in the reference's triplet order (sg.cpp:203-217).
__device__ __forceinline__ double transient_entry(const double* Kl_s, const double* Ml_s, int nl, int nin,
                                                  int lid, int nb, int dir, int kt, int jt, int nt, double ms,
                                                  double ss, const int* gp_ptr, const int* gp_i,
                                                  const double* gp_v) {
  double v = (kt == jt) ? ms * mcoef(Ml_s, nl, lid, nb, dir) : 0.0;
  if (dir >= 5) return v;
  const int pr = kt * nt + jt;
  for (int e = gp_ptr[pr]; e < gp_ptr[pr + 1]; ++e) {
    const int i = gp_i[e];
    v += (ss * gp_v[e]) * kcoef(Kl_s + (size_t)i * 3 * nl, nl, lid, nb, dir);
  }
  return v;
}

struct SetupArgs {
  const double *Kl, *Ml;
  const int *gp_ptr, *gp_i;
  const double* gp_v;
  const int* lid_to_p;
  const int* ng;
  int nl, nin, nt, mx, my, W, H, B;
  double ms, ss;
};

// D_k (same grid row) and E_k (row k+1 to row k) blocks; thread per (s, k, row).
__global__ void assemble_ii_kernel(SetupArgs A, double* __restrict__ D, double* __restrict__ E, int ns) {
  const long long total = (long long)ns * A.H * A.B;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int row = int(t % A.B), k = int((t / A.B) % A.H), s = int(t / ((long long)A.B * A.H));
    const int i = row / A.nt, kt = row % A.nt;
    const int il = i + 1, jl = k + 1, lid = jl * (A.mx + 1) + il;
    const double* Kl_s = A.Kl + (size_t)s * A.nin * 3 * A.nl;
    const double* Ml_s = A.Ml + (size_t)s * 4 * A.nl;
    const int* cls = A.lid_to_p + (size_t)s * A.nl;
    double* Dk = D + ((size_t)s * A.H + k) * A.B * A.B;
    // positions of the padded grid that are not interior nodes of a ragged
    // block (its interface / boundary line, padding) are decoupled unit rows
    if (cls[lid] != -2) {
      Dk[(size_t)row * A.B + row] = 1.0;
      continue;
    }
    // same grid row: W, self, E
    for (int dir = 0; dir < 3; ++dir) {
      const int i2 = i + kDI[dir];
      if (i2 < 0 || i2 >= A.W) continue;
      const int nb = lid + kDI[dir];
      if (cls[nb] != -2) continue;
      for (int jt = 0; jt < A.nt; ++jt)
        Dk[(size_t)(i2 * A.nt + jt) * A.B + row] =
            transient_entry(Kl_s, Ml_s, A.nl, A.nin, lid, nb, dir, kt, jt, A.nt, A.ms, A.ss, A.gp_ptr, A.gp_i, A.gp_v);
    }
    // E_{k-1}: this row (grid row k) against grid row k-1: S and SW neighbours
    if (k > 0) {
      double* Ek = E + ((size_t)s * (A.H - 1) + (k - 1)) * A.B * A.B;
      for (int dir : {4, 6}) {
        const int i2 = i + kDI[dir];
        if (i2 < 0) continue;
        const int nb = lid + kDI[dir] + kDJ[dir] * (A.mx + 1);
        if (cls[nb] != -2) continue;
        for (int jt = 0; jt < A.nt; ++jt)
          Ek[(size_t)(i2 * A.nt + jt) * A.B + row] =
              transient_entry(Kl_s, Ml_s, A.nl, A.nin, lid, nb, dir, kt, jt, A.nt, A.ms, A.ss, A.gp_ptr, A.gp_i, A.gp_v);
      }
    }
  }
}

// R_k = rows of grid row k of A_IG (B x amax column-major per subdomain).
__global__ void assemble_rhs_kernel(SetupArgs A, int k, double* __restrict__ R, int amax, int ns) {
  const long long total = (long long)ns * A.B;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int row = int(t % A.B), s = int(t / A.B);
    const int i = row / A.nt, kt = row % A.nt;
    const int il = i + 1, jl = k + 1, lid = jl * (A.mx + 1) + il;
    const double* Kl_s = A.Kl + (size_t)s * A.nin * 3 * A.nl;
    const double* Ml_s = A.Ml + (size_t)s * 4 * A.nl;
    double* Rs = R + (size_t)s * A.B * amax;
    const int ng = A.ng[s];
    if (A.lid_to_p[(size_t)s * A.nl + lid] != -2) continue;  // unit row of a ragged block
    for (int dir = 1; dir < 7; ++dir) {
      const int nb = lid + kDI[dir] + kDJ[dir] * (A.mx + 1);
      const int p = A.lid_to_p[(size_t)s * A.nl + nb];
      if (p < 0) continue;
      for (int jt = 0; jt < A.nt; ++jt)
        Rs[(size_t)(jt * ng + p) * A.B + row] =
            transient_entry(Kl_s, Ml_s, A.nl, A.nin, lid, nb, dir, kt, jt, A.nt, A.ms, A.ss, A.gp_ptr, A.gp_i, A.gp_v);
    }
  }
}

// A_GG into S (amax x amax per subdomain); thread per (s, interface flat row).
__global__ void assemble_gg_kernel(SetupArgs A, const int* __restrict__ ip_off, const int* __restrict__ iface_lid,
                                   double* __restrict__ S, int amax, int ns) {
  const int s = blockIdx.y;
  const int ng = A.ng[s], a = ng * A.nt;
  const double* Kl_s = A.Kl + (size_t)s * A.nin * 3 * A.nl;
  const double* Ml_s = A.Ml + (size_t)s * 4 * A.nl;
  double* Ss = S + (size_t)s * amax * amax;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < a; f += gridDim.x * blockDim.x) {
    const int kt = f / ng, p = f % ng;
    const int lid = iface_lid[ip_off[s] + p];
    const int il = lid % (A.mx + 1), jl = lid / (A.mx + 1);
    for (int dir = 0; dir < 7; ++dir) {
      const int il2 = il + kDI[dir], jl2 = jl + kDJ[dir];
      if (il2 < 0 || il2 > A.mx || jl2 < 0 || jl2 > A.my) continue;
      const int nb = jl2 * (A.mx + 1) + il2;
      const int q = A.lid_to_p[(size_t)s * A.nl + nb];
      if (q < 0) continue;
      for (int jt = 0; jt < A.nt; ++jt)
        Ss[(size_t)(jt * ng + q) * amax + f] =
            transient_entry(Kl_s, Ml_s, A.nl, A.nin, lid, nb, dir, kt, jt, A.nt, A.ms, A.ss, A.gp_ptr, A.gp_i, A.gp_v);
    }
  }
}

__global__ void set_identity_kernel(double* X, int B, int count) {
  const long long total = (long long)count * B * B;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long e = t % ((long long)B * B);
    X[t] = (e / B == e % B) ? 1.0 : 0.0;
  }
}

// Sub-matrix gather: out(a, b) = S(ri[a], ci[b]) (column-major, ld_out = nrow)
__global__ void extract_kernel(const double* __restrict__ S, int lds, const int* __restrict__ ri, int nrow,
                               const int* __restrict__ ci, int ncol, double* __restrict__ out) {
  const long long total = (long long)nrow * ncol;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int a = int(t % nrow), b = int(t / nrow);
    out[t] = S[(size_t)ci[b] * lds + ri[a]];
  }
}

__global__ void add_diag_kernel(double* A, int n, int lda, double shift) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) A[(size_t)i * lda + i] += shift;
}
__global__ void symmetrize_lower_kernel(double* A, int n) {
  const long long total = (long long)n * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int r = int(t % n), c = int(t / n);
    if (r < c) A[t] = A[(size_t)r * n + c];
  }
}

namespace {
double diag_trace_host(const double* dA, int n, int lda, cudaStream_t st) {
  std::vector<double> h((size_t)n * lda);
  SGW_CUDA(cudaMemcpyAsync(h.data(), dA, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  SGW_CUDA(cudaStreamSynchronize(st));
  double tr = 0;
  for (int i = 0; i < n; ++i) tr += h[(size_t)i * lda + i];
  return tr;
}

}  // namespace

// llt_regularized (src/dd.cpp:66-76) followed by the inverse: A <- A^-1 (full).
void spd_inverse(cusolverDnHandle_t sol, cudaStream_t st, double* A, int n, DBuf<double>& work, DBuf<int>& info,
                 const char* what) {
  if (n == 0) return;
  std::vector<double> backup((size_t)n * n);
  SGW_CUDA(cudaMemcpyAsync(backup.data(), A, backup.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  int lw1 = 0, lw2 = 0;
  SGW_SOLVER(cusolverDnDpotrf_bufferSize(sol, CUBLAS_FILL_MODE_LOWER, n, A, n, &lw1));
  SGW_SOLVER(cusolverDnDpotri_bufferSize(sol, CUBLAS_FILL_MODE_LOWER, n, A, n, &lw2));
  if ((size_t)std::max(lw1, lw2) > work.n) work.alloc(std::max(lw1, lw2));
  SGW_SOLVER(cusolverDnDpotrf(sol, CUBLAS_FILL_MODE_LOWER, n, A, n, work.p, (int)work.n, info.p));
  int h = 0;
  SGW_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  SGW_CUDA(cudaStreamSynchronize(st));
  if (h != 0) {
    double tr = 0;
    for (int i = 0; i < n; ++i) tr += backup[(size_t)i * n + i];
    for (int i = 0; i < n; ++i) backup[(size_t)i * n + i] += 1e-10 * tr / n;
    SGW_CUDA(cudaMemcpyAsync(A, backup.data(), backup.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    SGW_SOLVER(cusolverDnDpotrf(sol, CUBLAS_FILL_MODE_LOWER, n, A, n, work.p, (int)work.n, info.p));
    SGW_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    SGW_CUDA(cudaStreamSynchronize(st));
    if (h != 0) throw Error(2, std::string("llt_regularized: factorization failed after regularization (") + what + ")");
  }
  SGW_SOLVER(cusolverDnDpotri(sol, CUBLAS_FILL_MODE_LOWER, n, A, n, work.p, (int)work.n, info.p));
  symmetrize_lower_kernel<<<cdiv((long long)n * n, 256), 256, 0, st>>>(A, n);
  SGW_LAUNCHED();
}
namespace {
}  // namespace

// ------------------------------------------------------------------ maps ---
void GpuSolver::build_maps() {
  const int ns = NS, nt = NT;
  ng_.resize(ns);
  nr_.resize(ns);
  nc_.resize(ns);
  std::vector<int> ipo(ns + 1, 0), cpo(ns + 1, 0), ipos, lidp, ilid, pk, cpos;
  std::vector<double> w;
  for (int s = 0; s < ns; ++s) {
    const auto& sd = G.sub[s];
    ng_[s] = int(sd.iface_lid.size());
    nr_[s] = int(sd.r_local.size());
    nc_[s] = int(sd.c_local.size());
    ipo[s + 1] = ipo[s] + ng_[s];
    cpo[s + 1] = cpo[s] + nc_[s];
    ipos.insert(ipos.end(), sd.iface_pos.begin(), sd.iface_pos.end());
    ilid.insert(ilid.end(), sd.iface_lid.begin(), sd.iface_lid.end());
    w.insert(w.end(), sd.w.begin(), sd.w.end());
    lidp.insert(lidp.end(), sd.lid_to_p.begin(), sd.lid_to_p.end());
    std::vector<int> kind(ng_[s], 0);
    for (int r = 0; r < nr_[s]; ++r) kind[sd.r_local[r]] = r;
    for (int c = 0; c < nc_[s]; ++c) kind[sd.c_local[c]] = -1 - c;
    pk.insert(pk.end(), kind.begin(), kind.end());
    cpos.insert(cpos.end(), sd.corner_pos.begin(), sd.corner_pos.end());
  }
  ip_off.upload(ipo);
  cp_off_.upload(cpo);
  iface_pos.upload(ipos);
  iface_w.upload(w);
  lid_to_p.upload(lidp);
  pkind_.upload(pk);
  cpos_flat_.upload(cpos);
  iface_lid_.upload(ilid);
  ng_d.upload(ng_);
  nr_d.upload(nr_);
  nc_d.upload(nc_);
  // node lists of the per-step coupling kernels: interface nodes, and interior
  // nodes with an interface neighbour (7-point pattern incl. NE / SW)
  {
    std::vector<int> il, al;
    const int w = G.mx + 1;
    for (int s = 0; s < ns; ++s) {
      const auto& sd = G.sub[s];
      for (int lid : sd.iface_lid) il.push_back(s * G.nl + lid);
      for (int lid = 0; lid < G.nl; ++lid) {
        if (sd.lid_to_p[lid] != -2) continue;
        const int i0 = lid % w, j0 = lid / w;
        bool adj = false;
        for (int dj = -1; dj <= 1 && !adj; ++dj)
          for (int di = -1; di <= 1 && !adj; ++di) {
            const int i2 = i0 + di, j2 = j0 + dj;
            if ((di == 1 && dj == -1) || (di == -1 && dj == 1)) continue;  // no NW / SE couplings
            if (i2 < 0 || j2 < 0 || i2 >= w || j2 >= G.my + 1) continue;
            adj = sd.lid_to_p[j2 * w + i2] >= 0;
          }
        if (adj) al.push_back(s * G.nl + lid);
      }
    }
    ilist_.upload(il), alist_.upload(al);
    n_ilist_ = (long long)il.size(), n_alist_ = (long long)al.size();
  }
  // inverse maps, ascending s (fixed reduction order of src/dd.cpp:151-155)
  std::vector<int> icnt(G.n_iface, 0), is(4 * G.n_iface, 0), ip(4 * G.n_iface, 0);
  std::vector<int> ccnt(G.n_corner, 0), cs(4 * std::max(1, G.n_corner), 0), cc(4 * std::max(1, G.n_corner), 0);
  for (int s = 0; s < ns; ++s) {
    const auto& sd = G.sub[s];
    for (int p = 0; p < ng_[s]; ++p) {
      const int g = sd.iface_pos[p];
      is[4 * g + icnt[g]] = s;
      ip[4 * g + icnt[g]] = p;
      ++icnt[g];
    }
    for (int c = 0; c < nc_[s]; ++c) {
      const int g = sd.corner_pos[c];
      cs[4 * g + ccnt[g]] = s;
      cc[4 * g + ccnt[g]] = c;
      ++ccnt[g];
    }
  }
  inv_cnt.upload(icnt);
  inv_s.upload(is);
  inv_p.upload(ip);
  cinv_cnt.upload(ccnt);
  cinv_s.upload(cs);
  cinv_c.upload(cc);
  std::vector<int> iod(n, -1);
  for (int q = 0; q < G.n_iface; ++q) iod[G.iface_dofs[q]] = q;
  iface_of_dof.upload(iod);
  // NN2 gathers: r-space padded like Qp (offsets set in setup_nn2), c-space compact
  coff_.assign(ns + 1, 0);
  for (int s = 0; s < ns; ++s) coff_[s + 1] = coff_[s] + (long long)nt * nc_[s];
  std::vector<int> cg(coff_[ns]);
  std::vector<double> cw(coff_[ns]);
  for (int s = 0; s < ns; ++s) {
    const auto& sd = G.sub[s];
    for (int j = 0; j < nt; ++j)
      for (int c = 0; c < nc_[s]; ++c) {
        const long long k = coff_[s] + (long long)j * nc_[s] + c;
        cg[k] = j * G.n_iface + sd.iface_pos[sd.c_local[c]];
        cw[k] = sd.w[sd.c_local[c]];
      }
  }
  c_gidx.upload(cg);
  c_w.upload(cw);
  d_coff.upload(coff_);
  sub_gid_d_.upload(G.sub_gid);
  gid_local_d_.upload(G.gid_to_local);
  build_halo();
}

// ---------------------------------------------------------- constructor ----
GpuSolver::GpuSolver(Problem p, std::unique_ptr<Comm> comm) : P(std::move(p)), comm_(std::move(comm)) {
  const auto t0 = std::chrono::steady_clock::now();
  const long long bytes0 = DevBytes::total.load();
  if ((int)P.coeff.size() != P.n_in * P.n_nodes() || P.n_in != P.tensor.n_in)
    throw Error(1, "SgSolver: coefficient terms do not match tensor input size");
  if (P.tensor.n_out < 1) throw Error(1, "SgSolver: tensor has no output terms");
  if (!(P.dt > 0.0)) throw Error(1, "SgSolver: dt must be positive");
  if (comm_ && (comm_->rank() != P.rank || comm_->size() != P.world)) throw Error(1, "communicator / rank mismatch");
  G = build_geometry(P.nx, P.ny, P.px, P.py, P.rank, P.world);
  // one subdomain (sg.cpp:146 direct_): no interface; the step's interior
  // solve is then the whole (P+1) n system (the reference's direct_llt_,
  // sg.cpp:158-172, :301-305) and the interface PCG is empty (0 iterations)
  if (G.ns_total >= 2 && G.n_iface == 0) throw Error(1, "partition without an interface");
  direct_ = G.n_iface_global == 0;
  NT = P.tensor.n_out;
  NIN = P.n_in;
  NS = G.ns;
  n = G.n;
  NG = NT * G.n_iface;
  NGG = (long long)NT * G.n_iface_global;
  NC = NT * G.n_corner;
  NSTATE = size_t(NT) * n;
  SGW_CUDA(cudaSetDevice(P.device));
  SGW_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  own_stream_ = true;
  for (auto& e : ev_) SGW_CUDA(cudaEventCreate(&e));
  SGW_CUDA(cudaMallocHost(&h_scal_, 8 * sizeof(double)));
  if (cublasCreate(&blas_) != CUBLAS_STATUS_SUCCESS) throw Error(4, "cublasCreate failed");
  if (cusolverDnCreate(&sol_) != CUSOLVER_STATUS_SUCCESS) throw Error(4, "cusolverDnCreate failed");
  cublasSetStream(blas_, st_);
  cusolverDnSetStream(sol_, st_);
  const double mf = 1.0 / (P.zeta * P.dt * P.dt), df = P.gamma / (P.zeta * P.dt);  // newmark.hpp:16-18
  P.mass_scale = mf + df * P.alpha0;
  P.stiff_scale = 1.0 + df * P.alpha1;

  // SGW_SETUP_TIMING=1: wall-clock phases of the constructor on stderr
  const bool timing = std::getenv("SGW_SETUP_TIMING") != nullptr;
  auto tlast = std::chrono::steady_clock::now();
  nvtxRangePushA("sgw setup");
  auto lap = [&](const char* what) {
    nvtxMarkA(what);
    if (!timing) return;
    cudaStreamSynchronize(st_);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[sgw setup] %-28s %8.3f s\n", what, std::chrono::duration<double>(now - tlast).count());
    tlast = now;
  };
  lap("handles");
  const Stencils stc = build_stencils(P, G, true);
  lap("build_stencils (host)");
  build_device_inputs(stc);
  lap("device inputs + SG-op JIT");
  build_maps();
  lap("build_maps");
  // setup in batches of subdomains sized so the dense temporaries (A_II block
  // factor, L^-1 blocks, S_s, the rolling L^-1 A_IG) stay within ~24 GB
  B = G.W * NT;
  amax_ = 0;
  for (int s = 0; s < NS; ++s) amax_ = std::max(amax_, NT * ng_[s]);
  if (!direct_) plan_nn2();
  build_sweep_layout();
  lap("plan_nn2 + sweep layout");
  {
    const double per = 8.0 * (3.0 * G.H * double(B) * B + double(amax_) * amax_ + 2.0 * double(B) * amax_);
    int nb = std::max(1, std::min(NS, int(24e9 / per)));
    if (const char* e = std::getenv("SGW_SETUP_BATCH")) nb = std::max(1, std::atoi(e));  // test hook
    std::vector<double> fcc((size_t)NC * NC, 0.0);
    for (int b0 = 0; b0 < NS; b0 += nb) {
      const int cnt = std::min(nb, NS - b0);
      setup_interior_and_schur(b0, cnt);
      lap("interior factor + Schur batch");
      if (!direct_) nn2_batch(b0, cnt, fcc);
      lap("NN2 batch");
    }
    if (!direct_) finish_nn2(fcc);
    lap("finish_nn2");
  }

  // work vectors (the step kernels use 32-bit index arithmetic)
  if (NSTATE >= (size_t(1) << 31) || (size_t)NS * G.H * B >= (size_t(1) << 31))
    throw Error(1, "state too large for one GPU (2^31 entries)");
  for (DBuf<double>* b : {&u, &v, &a, &um, &uc, &unext}) b->alloc(NSTATE), b->zero(st_);
  for (DBuf<double>* b : {&vb, &vx, &vr, &vz, &vp, &vq, &vrt}) b->alloc(NG), b->zero(st_);
  li_x.alloc(Sp.xlen), li_x.zero(st_);
  li_y.alloc(Sp.xlen), li_y.zero(st_);
  fG.alloc(Sp.xlen), fG.zero(st_);
  const size_t nI = size_t(NS) * G.H * B;
  fI.alloc(nI), yI.alloc(nI), wI.alloc(nI);
  yI.zero(st_), wI.zero(st_);  // unit rows of ragged blocks stay zero
  scal.alloc(16), scal.zero(st_);
  dpart.alloc(1024), dcount.alloc(4), dcount.zero(st_);
  lap("work vectors");
  setup_fused_pcg();
  lap("persistent PCG setup");
  build_coupling_blocks();  // A_GI / A_IG and interface-row force blocks, memory permitting
  lap("coupling blocks");
  SGW_CUDA(cudaStreamSynchronize(st_));
  nvtxRangePop();
  setup_bytes_ = DevBytes::total.load() - bytes0;
  setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void destroy_sweep_layout(SweepLayout* p);

GpuSolver::~GpuSolver() {
  destroy_sweep_layout(sweep_layout_);
  if (blas_) cublasDestroy(blas_);
  if (sol_) cusolverDnDestroy(sol_);
  for (auto& e : ev_) cudaEventDestroy(e);
  if (side_) cudaStreamDestroy(side_);
  if (graph_mv_) cudaGraphExecDestroy(graph_mv_);
  if (graph_pc_) cudaGraphExecDestroy(graph_pc_);
  if (h_scal_) cudaFreeHost(h_scal_);
  if (h_fused_) cudaFreeHost(h_fused_);
  if (h_st_) cudaFreeHost(h_st_);
  for (auto& ge : ph_graph_)
    if (ge) cudaGraphExecDestroy(ge);
  if (own_stream_ && st_) cudaStreamDestroy(st_);
}

void GpuSolver::set_stream(cudaStream_t s) {
  SGW_CUDA(cudaStreamSynchronize(st_));
  if (own_stream_) cudaStreamDestroy(st_);
  own_stream_ = s == nullptr;
  if (s == nullptr) SGW_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  st_ = s;
  cublasSetStream(blas_, st_);
  cusolverDnSetStream(sol_, st_);
}

void GpuSolver::build_device_inputs(const Stencils& stc) {
  // tensor lists from for_each (pce.hpp:34-39): both (j,k) and (k,j)
  struct E3 {
    int i, j, k;
    double v;
  };
  std::vector<E3> all;
  const TensorHost& t = P.tensor;
  for (size_t e = 0; e < t.v.size(); ++e) {
    if (t.i[e] < 0 || t.i[e] >= NIN || t.j[e] < 0 || t.k[e] < 0 || t.j[e] >= NT || t.k[e] >= NT)
      throw Error(1, "tensor entry out of range");
    all.push_back({t.i[e], t.j[e], t.k[e], t.v[e]});
    if (t.j[e] != t.k[e]) all.push_back({t.i[e], t.k[e], t.j[e], t.v[e]});
  }
  // by output term k: (i, j, g), ascending i (for_each order)
  std::stable_sort(all.begin(), all.end(), [](const E3& a, const E3& b) { return a.i < b.i; });
  std::vector<int> kptr(NT + 1, 0), ki, kj, pptr(NT * NT + 1, 0), pi;
  std::vector<double> kv, pv;
  for (const E3& e : all) kptr[e.k + 1]++;
  for (int k = 0; k < NT; ++k) kptr[k + 1] += kptr[k];
  ki.resize(all.size()), kj.resize(all.size()), kv.resize(all.size());
  {
    std::vector<int> fill(kptr.begin(), kptr.end() - 1);
    for (const E3& e : all) {
      const int pos = fill[e.k]++;
      ki[pos] = e.i, kj[pos] = e.j, kv[pos] = e.v;
    }
  }
  // by pair (row term k, col term j): (i, g)
  for (const E3& e : all) pptr[e.k * NT + e.j + 1]++;
  for (int q = 0; q < NT * NT; ++q) pptr[q + 1] += pptr[q];
  pi.resize(all.size()), pv.resize(all.size());
  {
    std::vector<int> fill(pptr.begin(), pptr.end() - 1);
    for (const E3& e : all) {
      const int pos = fill[e.k * NT + e.j]++;
      pi[pos] = e.i, pv[pos] = e.v;
    }
  }
  gk_ptr.upload(kptr), gk_i.upload(ki), gk_j.upload(kj), gk_v.upload(kv);
  gp_ptr.upload(pptr), gp_i.upload(pi), gp_v.upload(pv);
  Kg.upload(stc.Kg), Mg.upload(stc.Mg), Kl.upload(stc.Kl), Ml.upload(stc.Ml);
  // JIT SG operator (sgop.cu) on the global grid, couplings stored strip by strip
  sgop_ = build_sgop(NT, NIN, P.tensor);
  if (sgop_) {
    std::vector<double> kt;
    SgOpArgs& a = sgop_args_;
    if (!sgop_pack_stencils(*sgop_, stc.Kg.data(), stc.Mg.data(), P.nx - 1, P.ny - 1, NIN, kt, a)) {
      sgop_.reset();  // non-constant mass stencil: the table-driven kernel
    } else {
      Kp_.upload(kt);
      Kpart_.alloc(sgop_scratch_doubles(*sgop_, P.nx - 1, P.ny - 1));
      a.K = Kp_.p, a.part = Kpart_.p;
      a.xterm = a.yterm = n;
      a.xpitch = a.ypitch = P.nx - 1;
    }
  }
  if (sgop_) {
    yglob_.alloc(NSTATE);
  }
}

// -------------------------------------------------- interior and Schur -----
// Subdomains [b0, b0 + nb): dense per-batch temporaries (block Cholesky of A_II,
// L^-1 blocks, the local Schur S_s), then the factor tiles go to Fcomp and S_s
// to Sdense_ (batch-local) for nn2_batch.  Batched cuSOLVER / cuBLAS calls per
// grid row k over the batch.
void GpuSolver::setup_interior_and_schur(int b0, int nb) {
  const int H = G.H, W = G.W, ns = nb, amax = amax_;
  SetupArgs A{Kl.p + (size_t)b0 * NIN * 3 * G.nl, Ml.p + (size_t)b0 * 4 * G.nl, gp_ptr.p, gp_i.p, gp_v.p,
              lid_to_p.p + (size_t)b0 * G.nl, ng_d.p + b0, G.nl, NIN, NT, G.mx, G.my, W, H, B,
              P.mass_scale, P.stiff_scale};
  const size_t BB = size_t(B) * B;
  DBuf<double> D;
  D.alloc(size_t(ns) * H * BB);
  D.zero(st_);
  Lsub.alloc(size_t(ns) * std::max(0, H - 1) * BB);
  Lsub.zero(st_);
  {
    const long long tot = (long long)ns * H * B;
    assemble_ii_kernel<<<std::min(cdiv(tot, 256), 65535), 256, 0, st_>>>(A, D.p, Lsub.p, ns);
    SGW_LAUNCHED();
  }
  extract_band_batch(b0, nb);  // A_{k+1,k} band for the sweeps, before the factorization
  Linv.alloc(size_t(ns) * H * BB);
  set_identity_kernel<<<std::min(cdiv((long long)ns * H * BB, 256), 65535), 256, 0, st_>>>(Linv.p, B, ns * H);
  SGW_LAUNCHED();
  // pointer tables [k][s] for the batched calls
  std::vector<double*> hD(size_t(H) * ns), hL(size_t(H) * ns), hI(size_t(H) * ns);
  for (int k = 0; k < H; ++k)
    for (int q = 0; q < ns; ++q) {
      hD[size_t(k) * ns + q] = D.p + (size_t(q) * H + k) * BB;
      hL[size_t(k) * ns + q] = k < H - 1 ? Lsub.p + (size_t(q) * (H - 1) + k) * BB : nullptr;
      hI[size_t(k) * ns + q] = Linv.p + (size_t(q) * H + k) * BB;
    }
  DBuf<double*> pD, pL, pI;
  pD.upload(hD), pL.upload(hL), pI.upload(hI);
  // block Cholesky over grid rows (src/sg.cpp:218-225 restated block-wise)
  DBuf<int> info;
  info.alloc(size_t(ns) * H);
  info.zero(st_);
  const double one = 1.0, mone = -1.0;
  for (int k = 0; k < H; ++k) {
    if (k > 0)
      SGW_BLAS(cublasDgemmStridedBatched(blas_, CUBLAS_OP_N, CUBLAS_OP_T, B, B, B, &mone, Lsub.p + (k - 1) * BB, B,
                                         (long long)(H - 1) * BB, Lsub.p + (k - 1) * BB, B, (long long)(H - 1) * BB,
                                         &one, D.p + k * BB, B, (long long)H * BB, ns));
    SGW_SOLVER(cusolverDnDpotrfBatched(sol_, CUBLAS_FILL_MODE_LOWER, B, pD.p + size_t(k) * ns, B, info.p + size_t(k) * ns,
                                       ns));
    if (k < H - 1)
      SGW_BLAS(cublasDtrsmBatched(blas_, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, B,
                                  B, &one, pD.p + size_t(k) * ns, B, pL.p + size_t(k) * ns, B, ns));
  }
  {
    std::vector<int> h(info.n);
    SGW_CUDA(cudaMemcpyAsync(h.data(), info.p, h.size() * sizeof(int), cudaMemcpyDeviceToHost, st_));
    SGW_CUDA(cudaStreamSynchronize(st_));
    for (int k = 0; k < H; ++k)
      for (int q = 0; q < ns; ++q)
        if (h[size_t(k) * ns + q] != 0)
          throw Error(2, "stochastic interior factorization failed (subdomain " + std::to_string(G.sub_gid[b0 + q]) + ")");
  }
  // S_s = A_GG - Y^T Y, Y = L^-1 A_IG by rolling block forward substitution
  // (one subdomain, no interface: amax = 0, nothing to eliminate)
  if (amax > 0) {
  Sdense_.alloc(size_t(ns) * amax * amax);
  Sdense_.zero(st_);
  assemble_gg_kernel<<<dim3(cdiv(amax, 128), ns), 128, 0, st_>>>(A, ip_off.p + b0, iface_lid_.p, Sdense_.p, amax, ns);
  SGW_LAUNCHED();
  if (P.precond == 2)  // lumped: K~_GG before the elimination (det_loop.cpp:165-167, flattened)
    for (int q = 0; q < ns; ++q) pack_tiles_range(Aggp, b0 + q, Sdense_.p + size_t(q) * amax * amax, amax, st_);
  DBuf<double> R, Y;
  R.alloc(size_t(ns) * B * amax);
  Y.alloc(size_t(ns) * B * amax);
  const long long sRY = (long long)B * amax, sS = (long long)amax * amax;
  std::vector<double*> hR(ns), hY(ns);
  for (int q = 0; q < ns; ++q) hR[q] = R.p + q * sRY, hY[q] = Y.p + q * sRY;
  DBuf<double*> pR, pY;
  pR.upload(hR), pY.upload(hY);
  for (int k = 0; k < H; ++k) {
    R.zero(st_);
    assemble_rhs_kernel<<<cdiv((long long)ns * B, 256), 256, 0, st_>>>(A, k, R.p, amax, ns);
    SGW_LAUNCHED();
    if (k > 0)
      SGW_BLAS(cublasDgemmStridedBatched(blas_, CUBLAS_OP_N, CUBLAS_OP_N, B, amax, B, &mone, Lsub.p + (k - 1) * BB, B,
                                         (long long)(H - 1) * BB, Y.p, B, sRY, &one, R.p, B, sRY, ns));
    SGW_BLAS(cublasDtrsmBatched(blas_, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, B,
                                amax, &one, pD.p + size_t(k) * ns, B, pR.p, B, ns));
    SGW_BLAS(cublasDgemmStridedBatched(blas_, CUBLAS_OP_T, CUBLAS_OP_N, amax, amax, B, &mone, R.p, B, sRY, R.p, B, sRY,
                                       &one, Sdense_.p, amax, sS, ns));
    std::swap(R.p, Y.p);
    std::swap(pR.p, pY.p);
  }
  R.reset();
  Y.reset();
  }
  // Linv_kk = L_kk^-1 (exact zeros above the diagonal) for the per-step sweeps
  for (int k = 0; k < H; ++k)
    SGW_BLAS(cublasDtrsmBatched(blas_, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, B, B,
                                &one, pD.p + size_t(k) * ns, B, pI.p + size_t(k) * ns, B, ns));
  // D_k^-1 = L_kk^-T L_kk^-1 (block Thomas form of the sweeps) over the finished factor blocks
  const double zero = 0.0;
  SGW_BLAS(cublasDgemmStridedBatched(blas_, CUBLAS_OP_T, CUBLAS_OP_N, B, B, B, &one, Linv.p, B, (long long)BB, Linv.p,
                                     B, (long long)BB, &zero, D.p, B, (long long)BB, ns * H));
  compact_dinv_batch(b0, nb, D.p);
  D.reset();
  Linv.reset();
  Lsub.reset();
}

// ------------------------------------------------------------ NN2 data -----
// src/dd.cpp:98-140: S_rr, S_rc, S_cc; Q = S_rr^-1 (explicit), Psi = Q S_rc,
// F_cc = sum_s B_s^T (S_cc - S_rc^T Psi) B_s assembled in ascending s.
void GpuSolver::plan_nn2() {
  const int ns = NS, nt = NT;
  std::vector<int> dimsS(ns), dimsQ(ns);
  for (int s = 0; s < ns; ++s) dimsS[s] = nt * ng_[s], dimsQ[s] = nt * nr_[s];
  Sp.plan(dimsS, !P.implicit_schur);  // reduced-memory mode: layout only, no S tiles
  Qp.plan(dimsQ);
  if (P.precond == 1) Sinvp.plan(dimsS);
  if (P.precond == 2) Aggp.plan(dimsS);
  roff_ = Qp.xoff;
  d_roff.upload(roff_);
  psioff_.assign(ns + 1, 0);
  for (int s = 0; s < ns; ++s) psioff_[s + 1] = psioff_[s] + (long long)nt * nr_[s] * nt * nc_[s];
  d_psioff.upload(psioff_);
  Psi.alloc(std::max<long long>(1, psioff_[ns]));
  // r-space gather map (padded like Qp)
  {
    std::vector<int> rg(Qp.xlen, -1);
    std::vector<double> rw(Qp.xlen, 0.0);
    for (int s = 0; s < ns; ++s) {
      const auto& sd = G.sub[s];
      for (int j = 0; j < nt; ++j)
        for (int r = 0; r < nr_[s]; ++r) {
          const long long k = roff_[s] + (long long)j * nr_[s] + r;
          rg[k] = j * G.n_iface + sd.iface_pos[sd.r_local[r]];
          rw[k] = sd.w[sd.r_local[r]];
        }
    }
    r_gidx.upload(rg);
    r_w.upload(rw);
  }
  r_x.alloc(Qp.xlen), r_x.zero(st_);
  r_t.alloc(Qp.xlen);
  c_f.alloc(std::max<long long>(1, coff_[ns])), c_d.alloc(std::max<long long>(1, coff_[ns]));
  dcoarse.alloc(std::max(1, NC)), ucoarse.alloc(std::max(1, NC));
  ucoarse.zero(st_);
}

// Subdomains [b0, b0 + nb) with S_s in Sdense_ (batch-local): S tiles, and per
// subdomain extract, invert, Psi, local coarse block (accumulated into fcc).
void GpuSolver::nn2_batch(int b0, int nb, std::vector<double>& fcc) {
  const int nt = NT, amax = amax_;
  if (!P.implicit_schur)
    for (int q = 0; q < nb; ++q) pack_tiles_range(Sp, b0 + q, Sdense_.p + size_t(q) * amax * amax, amax, st_);
  DBuf<double> Srr, Src, Scc, work;
  DBuf<int> ri, ci, info;
  info.alloc(1);
  const double one = 1.0, zero = 0.0, mone = -1.0;
  for (int s = b0; s < b0 + nb; ++s) {
    const auto& sd = G.sub[s];
    const int a = nt * ng_[s], rs = nt * nr_[s], cs = nt * nc_[s];
    std::vector<int> hr, hc;
    for (int j = 0; j < nt; ++j) {
      for (int r : sd.r_local) hr.push_back(j * ng_[s] + r);
      for (int c : sd.c_local) hc.push_back(j * ng_[s] + c);
    }
    ri.upload(hr);
    ci.upload(hc);
    const double* Ss = Sdense_.p + size_t(s - b0) * amax * amax;
    if (P.precond == 1 && a > 0) {  // NN1: llt_regularized(S_s) (dd.cpp:115) as an explicit inverse
      DBuf<double> Sf;
      Sf.alloc((size_t)a * a);
      SGW_CUDA(cudaMemcpy2DAsync(Sf.p, a * sizeof(double), Ss, amax * sizeof(double), a * sizeof(double), a,
                                 cudaMemcpyDeviceToDevice, st_));
      spd_inverse(sol_, st_, Sf.p, a, work, info, ("S of subdomain " + std::to_string(s)).c_str());
      pack_tiles_range(Sinvp, s, Sf.p, a, st_);
      SGW_CUDA(cudaStreamSynchronize(st_));
    }
    if (rs > 0) {
      Srr.alloc((size_t)rs * rs);
      extract_kernel<<<cdiv((long long)rs * rs, 256), 256, 0, st_>>>(Ss, amax, ri.p, rs, ri.p, rs, Srr.p);
      SGW_LAUNCHED();
      spd_inverse(sol_, st_, Srr.p, rs, work, info, ("subdomain " + std::to_string(s)).c_str());
      pack_tiles_range(Qp, s, Srr.p, rs, st_);
    }
    if (cs > 0) {
      Scc.alloc((size_t)cs * cs);
      extract_kernel<<<cdiv((long long)cs * cs, 256), 256, 0, st_>>>(Ss, amax, ci.p, cs, ci.p, cs, Scc.p);
      SGW_LAUNCHED();
      if (rs > 0) {
        Src.alloc((size_t)rs * cs);
        extract_kernel<<<cdiv((long long)rs * cs, 256), 256, 0, st_>>>(Ss, amax, ri.p, rs, ci.p, cs, Src.p);
        SGW_LAUNCHED();
        double* Ps = Psi.p + psioff_[s];
        SGW_BLAS(cublasDsymm(blas_, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, rs, cs, &one, Srr.p, rs, Src.p, rs, &zero,
                             Ps, rs));
        SGW_BLAS(cublasDgemm(blas_, CUBLAS_OP_T, CUBLAS_OP_N, cs, cs, rs, &mone, Src.p, rs, Ps, rs, &one, Scc.p, cs));
      }
      std::vector<double> h((size_t)cs * cs);
      SGW_CUDA(cudaMemcpyAsync(h.data(), Scc.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st_));
      SGW_CUDA(cudaStreamSynchronize(st_));
      for (int b2 = 0; b2 < cs; ++b2)
        for (int a2 = 0; a2 < cs; ++a2) {
          const int ja = a2 / nc_[s], ca = a2 % nc_[s], jb = b2 / nc_[s], cb = b2 % nc_[s];
          const int ga = ja * G.n_corner + sd.corner_pos[ca], gb = jb * G.n_corner + sd.corner_pos[cb];
          fcc[(size_t)gb * NC + ga] += h[(size_t)b2 * cs + a2];
        }
    }
  }
  Sdense_.reset();
}

void GpuSolver::finish_nn2(std::vector<double>& fcc) {
  DBuf<double> work;
  DBuf<int> info;
  info.alloc(1);
  if (NC > 0 && comm_) {  // F_cc = sum over all ranks' subdomains (dd.cpp:128-137)
    Finv.upload(fcc);
    allreduce(Finv.p, fcc.size());
    SGW_CUDA(cudaMemcpyAsync(fcc.data(), Finv.p, fcc.size() * sizeof(double), cudaMemcpyDeviceToHost, st_));
    SGW_CUDA(cudaStreamSynchronize(st_));
  }
  if (comm_ && comm_->solo())  // one rank alone: corners no owned subdomain touches get a unit row
    for (int c = 0; c < NC; ++c)
      if (fcc[(size_t)c * NC + c] == 0.0) fcc[(size_t)c * NC + c] = 1.0;
  fcc_host_ = fcc;
  if (NC > 0) {
    Finv.upload(fcc);
    spd_inverse(sol_, st_, Finv.p, NC, work, info, "coarse F_cc");
  }
  SGW_CUDA(cudaStreamSynchronize(st_));
}

}  // namespace sgw
