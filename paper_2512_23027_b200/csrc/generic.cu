// Interface systems built from caller-supplied local Schur data, and the PCG
// of src/pcg.cpp:7-50 over arbitrary operators.
//
// The structured-mesh solver (setup.cu, pcg_fused.cu) derives its S_s tiles
// from the partition.  These entry points take the reference's LocalSchur
// fields directly (include/sgwave/dd.hpp:50-62: S, gmap, weights, r_idx,
// c_idx, corner_gmap), as test_dd.cpp:123-151 builds one by hand, and run
// SchurSystem::finalize / matvec / apply_nn2 (src/dd.cpp:98-157, :199-253) on
// the device: dense S_s, explicit S_rr^-1 and F_cc^-1 from cuSOLVER
// (llt_regularized's shift-and-retry, src/dd.cpp:66-76), cuBLAS products, and
// gather / scatter kernels applied local by local in a fixed order (bitwise
// reproducible).  Sizes are those of unit tests and small systems; the
// production path is the tiled one.
#include "generic.cuh"

#include <algorithm>
#include <cmath>

namespace sgw {

namespace {
#define SGW_BLAS(call)                                                       \
  do {                                                                       \
    if ((call) != CUBLAS_STATUS_SUCCESS) throw Error(4, "cuBLAS failure: " #call); \
  } while (0)

__global__ void gather_w_kernel(const double* __restrict__ x, const long long* __restrict__ map,
                                const double* __restrict__ w, int n, double* __restrict__ out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    out[k] = w ? x[map[k]] * w[k] : x[map[k]];
}
__global__ void gather_i_kernel(const double* __restrict__ x, const int* __restrict__ idx, int n,
                                double* __restrict__ out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) out[k] = x[idx[k]];
}
__global__ void put_i_kernel(const double* __restrict__ v, const int* __restrict__ idx, int n, double* __restrict__ out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) out[idx[k]] = v[k];
}
// out[map[k]] += (w ? w[k] : 1) v[k]; map is injective within one local
__global__ void scatter_add_kernel(const double* __restrict__ v, const long long* __restrict__ map,
                                   const double* __restrict__ w, int n, double* __restrict__ out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    out[map[k]] += w ? v[k] * w[k] : v[k];
}
int grid_of(long long n) { return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 1024)); }
}  // namespace

// A <- A^-1 (SPD, column-major, device): setup.cu's spd_inverse, i.e.
// llt_regularized (src/dd.cpp:66-76) then the explicit inverse
void spd_inverse_inplace(cusolverDnHandle_t sol, cudaStream_t st, double* A, int n) {
  DBuf<double> work;
  DBuf<int> info;
  info.alloc(1);
  spd_inverse(sol, st, A, n, work, info, "local Schur");
}

GenericSchur::GenericSchur(long long n_global, long long n_corner, const std::vector<LocalInput>& in)
    : n_global_(n_global), n_corner_(n_corner) {
  SGW_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  if (cublasCreate(&blas_) != CUBLAS_STATUS_SUCCESS) throw Error(4, "cublasCreate failed");
  if (cusolverDnCreate(&sol_) != CUSOLVER_STATUS_SUCCESS) throw Error(4, "cusolverDnCreate failed");
  cublasSetStream(blas_, st_);
  cusolverDnSetStream(sol_, st_);
  if (n_global < 0 || n_corner < 0) throw Error(1, "schur_from_locals: negative sizes");
  fcc_.assign((size_t)n_corner * n_corner, 0.0);
  for (const LocalInput& li : in) {
    if (li.n < 0 || li.nr < 0 || li.nc < 0 || li.nr + li.nc > li.n) throw Error(1, "schur_from_locals: bad local sizes");
    for (int k = 0; k < li.n; ++k)
      if (li.gmap[k] < 0 || li.gmap[k] >= n_global) throw Error(1, "schur_from_locals: gmap out of range");
    for (int a = 0; a < li.nc; ++a)
      if (li.corner_gmap[a] < 0 || li.corner_gmap[a] >= n_corner)
        throw Error(1, "schur_from_locals: corner_gmap out of range");
    auto L = std::make_unique<Local>();
    L->n = li.n, L->nr = li.nr, L->nc = li.nc;
    L->S.upload(std::vector<double>(li.S, li.S + (size_t)li.n * li.n));
    L->w.upload(std::vector<double>(li.weights, li.weights + li.n));
    L->gmap.upload(std::vector<long long>(li.gmap, li.gmap + li.n));
    L->ridx.upload(std::vector<int>(li.r_idx, li.r_idx + li.nr));
    L->cidx.upload(std::vector<int>(li.c_idx, li.c_idx + li.nc));
    L->cgmap.upload(std::vector<long long>(li.corner_gmap, li.corner_gmap + li.nc));
    // S_rr^-1 and S_rc from S (src/dd.cpp:109-121); host extraction (setup)
    std::vector<double> srr((size_t)li.nr * li.nr), src((size_t)li.nr * li.nc), scc((size_t)li.nc * li.nc);
    auto S = [&](int a, int b) { return li.S[(size_t)b * li.n + a]; };
    for (int b = 0; b < li.nr; ++b)
      for (int a = 0; a < li.nr; ++a) srr[(size_t)b * li.nr + a] = S(li.r_idx[a], li.r_idx[b]);
    for (int b = 0; b < li.nc; ++b)
      for (int a = 0; a < li.nr; ++a) src[(size_t)b * li.nr + a] = S(li.r_idx[a], li.c_idx[b]);
    for (int b = 0; b < li.nc; ++b)
      for (int a = 0; a < li.nc; ++a) scc[(size_t)b * li.nc + a] = S(li.c_idx[a], li.c_idx[b]);
    L->Srr_inv.upload(srr);
    L->Src.upload(src);
    spd_inverse_inplace(sol_, st_, L->Srr_inv.p, li.nr);
    // coarse contribution S_cc - S_rc^T S_rr^-1 S_rc (src/dd.cpp:122-137)
    if (li.nc > 0 && n_corner > 0) {
      if (li.nr > 0) {
        DBuf<double> t, c;
        t.alloc((size_t)li.nr * li.nc), c.upload(scc);
        const double one = 1.0, zero = 0.0, mone = -1.0;
        SGW_BLAS(cublasDgemm(blas_, CUBLAS_OP_N, CUBLAS_OP_N, li.nr, li.nc, li.nr, &one, L->Srr_inv.p, li.nr, L->Src.p,
                             li.nr, &zero, t.p, li.nr));
        SGW_BLAS(cublasDgemm(blas_, CUBLAS_OP_T, CUBLAS_OP_N, li.nc, li.nc, li.nr, &mone, L->Src.p, li.nr, t.p, li.nr,
                             &one, c.p, li.nc));
        SGW_CUDA(cudaMemcpyAsync(scc.data(), c.p, scc.size() * 8, cudaMemcpyDeviceToHost, st_));
        SGW_CUDA(cudaStreamSynchronize(st_));
      }
      for (int a = 0; a < li.nc; ++a)
        for (int b = 0; b < li.nc; ++b)
          fcc_[(size_t)li.corner_gmap[b] * n_corner + li.corner_gmap[a]] += scc[(size_t)b * li.nc + a];
    }
    maxn_ = std::max(maxn_, li.n);
    locals_.push_back(std::move(L));
    tloc_.emplace_back();
    tloc_.back().alloc(std::max(1, li.nr));
  }
  if (n_corner > 0) {
    Finv_.upload(fcc_);
    spd_inverse_inplace(sol_, st_, Finv_.p, (int)n_corner);
  }
  xl_.alloc(std::max(1, maxn_)), yl_.alloc(std::max(1, maxn_)), t_.alloc(std::max(1, maxn_) * 2);
  d_.alloc(std::max<long long>(1, n_corner)), uc_.alloc(std::max<long long>(1, n_corner));
  SGW_CUDA(cudaStreamSynchronize(st_));
}

GenericSchur::~GenericSchur() {
  if (blas_) cublasDestroy(blas_);
  if (sol_) cusolverDnDestroy(sol_);
  if (st_) cudaStreamDestroy(st_);
}

// y = sum_s R_s^T S_s R_s x (src/dd.cpp:142-157)
void GenericSchur::matvec(const double* x, double* y) {
  SGW_CUDA(cudaMemsetAsync(y, 0, std::max<long long>(1, n_global_) * 8, st_));
  const double one = 1.0, zero = 0.0;
  for (auto& L : locals_) {
    if (L->n == 0) continue;
    gather_w_kernel<<<grid_of(L->n), 256, 0, st_>>>(x, L->gmap.p, nullptr, L->n, xl_.p);
    SGW_BLAS(cublasDgemv(blas_, CUBLAS_OP_N, L->n, L->n, &one, L->S.p, L->n, xl_.p, 1, &zero, yl_.p, 1));
    scatter_add_kernel<<<grid_of(L->n), 256, 0, st_>>>(yl_.p, L->gmap.p, nullptr, L->n, y);
    SGW_LAUNCHED();
  }
}

// z = sum_s R_s^T D_s [(R^r)^T S_rr^-1 R^r + coarse] D_s R_s r (src/dd.cpp:199-253)
void GenericSchur::apply_nn2(const double* r, double* z) {
  const double one = 1.0, zero = 0.0, mone = -1.0;
  SGW_CUDA(cudaMemsetAsync(z, 0, std::max<long long>(1, n_global_) * 8, st_));
  if (n_corner_ > 0) SGW_CUDA(cudaMemsetAsync(d_.p, 0, n_corner_ * 8, st_));
  // phase 1: t_s = S_rr^-1 (D r)_r, the coarse right-hand side d (kept per local)
  for (size_t s = 0; s < locals_.size(); ++s) {
    Local& L = *locals_[s];
    if (L.n == 0) continue;
    gather_w_kernel<<<grid_of(L.n), 256, 0, st_>>>(r, L.gmap.p, L.w.p, L.n, xl_.p);  // rl
    if (L.nr > 0) {
      gather_i_kernel<<<grid_of(L.nr), 256, 0, st_>>>(xl_.p, L.ridx.p, L.nr, yl_.p);
      SGW_BLAS(cublasDgemv(blas_, CUBLAS_OP_N, L.nr, L.nr, &one, L.Srr_inv.p, L.nr, yl_.p, 1, &zero, tloc_[s].p, 1));
    }
    if (L.nc > 0 && n_corner_ > 0) {
      gather_i_kernel<<<grid_of(L.nc), 256, 0, st_>>>(xl_.p, L.cidx.p, L.nc, t_.p);  // dc = rl_c
      if (L.nr > 0)  // dc -= S_rc^T t
        SGW_BLAS(cublasDgemv(blas_, CUBLAS_OP_T, L.nr, L.nc, &mone, L.Src.p, L.nr, tloc_[s].p, 1, &one, t_.p, 1));
      scatter_add_kernel<<<grid_of(L.nc), 256, 0, st_>>>(t_.p, L.cgmap.p, nullptr, L.nc, d_.p);
    }
    SGW_LAUNCHED();
  }
  if (n_corner_ > 0)  // u_c = F_cc^-1 d
    SGW_BLAS(cublasDgemv(blas_, CUBLAS_OP_N, (int)n_corner_, (int)n_corner_, &one, Finv_.p, (int)n_corner_, d_.p, 1,
                         &zero, uc_.p, 1));
  // phase 2: u_r = t - S_rr^-1 S_rc u_c; zl = [u_r | u_c] weighted, summed
  for (size_t s = 0; s < locals_.size(); ++s) {
    Local& L = *locals_[s];
    if (L.n == 0) continue;
    SGW_CUDA(cudaMemsetAsync(yl_.p, 0, L.n * 8, st_));
    if (L.nc > 0 && n_corner_ > 0) {
      gather_w_kernel<<<grid_of(L.nc), 256, 0, st_>>>(uc_.p, L.cgmap.p, nullptr, L.nc, t_.p);  // ucl
      if (L.nr > 0) {
        double* tmp = t_.p + maxn_;
        SGW_BLAS(cublasDgemv(blas_, CUBLAS_OP_N, L.nr, L.nc, &one, L.Src.p, L.nr, t_.p, 1, &zero, tmp, 1));
        SGW_BLAS(cublasDgemv(blas_, CUBLAS_OP_N, L.nr, L.nr, &mone, L.Srr_inv.p, L.nr, tmp, 1, &one, tloc_[s].p, 1));
      }
      put_i_kernel<<<grid_of(L.nc), 256, 0, st_>>>(t_.p, L.cidx.p, L.nc, yl_.p);
    }
    if (L.nr > 0) put_i_kernel<<<grid_of(L.nr), 256, 0, st_>>>(tloc_[s].p, L.ridx.p, L.nr, yl_.p);
    scatter_add_kernel<<<grid_of(L.n), 256, 0, st_>>>(yl_.p, L.gmap.p, L.w.p, L.n, z);
    SGW_LAUNCHED();
  }
}

// pcg (src/pcg.cpp:7-50) on device vectors of length n: x0 = 0, stop on the
// recurrence residual, confirm with the true residual b - A x (not counted as
// an iteration; the history records the true residual instead), restart from
// it (p kept) when the confirmation fails.
int pcg_generic(cublasHandle_t blas, cudaStream_t st, long long n, const DevOp& op, const DevOp& pre,
                const double* b, double* x, double tol, int max_iter, bool* converged, std::vector<double>* hist) {
  if (n > (1LL << 31) - 1) throw Error(1, "pcg: vector too long");
  const int m = (int)n;
  std::vector<double> h;
  DBuf<double> r, z, p, ap, rt;
  for (DBuf<double>* v : {&r, &z, &p, &ap, &rt}) v->alloc(std::max(1, m));
  SGW_CUDA(cudaMemsetAsync(x, 0, std::max(1, m) * 8, st));
  auto dot = [&](const double* a, const double* c) {
    double v = 0.0;
    SGW_BLAS(cublasDdot(blas, m, a, 1, c, 1, &v));  // host pointer mode: synchronous
    return v;
  };
  const double bnorm = std::sqrt(dot(b, b));
  int it = 0;
  *converged = false;
  if (bnorm == 0.0) {
    *converged = true;
    h.push_back(0.0);
  } else {
    SGW_CUDA(cudaMemcpyAsync(r.p, b, m * 8, cudaMemcpyDeviceToDevice, st));
    pre(r.p, z.p);
    SGW_CUDA(cudaMemcpyAsync(p.p, z.p, m * 8, cudaMemcpyDeviceToDevice, st));
    double rz = dot(r.p, z.p);
    h.push_back(1.0);
    for (; it < max_iter;) {
      op(p.p, ap.p);
      const double alpha = rz / dot(p.p, ap.p), malpha = -alpha;
      SGW_BLAS(cublasDaxpy(blas, m, &alpha, p.p, 1, x, 1));
      SGW_BLAS(cublasDaxpy(blas, m, &malpha, ap.p, 1, r.p, 1));
      ++it;
      double rel = std::sqrt(dot(r.p, r.p)) / bnorm;
      if (rel <= tol) {
        op(x, rt.p);  // r_true = b - A x
        const double mone = -1.0, one = 1.0;
        SGW_BLAS(cublasDscal(blas, m, &mone, rt.p, 1));
        SGW_BLAS(cublasDaxpy(blas, m, &one, b, 1, rt.p, 1));
        rel = std::sqrt(dot(rt.p, rt.p)) / bnorm;
        h.push_back(rel);
        if (rel <= tol) {
          *converged = true;
          break;
        }
        SGW_CUDA(cudaMemcpyAsync(r.p, rt.p, m * 8, cudaMemcpyDeviceToDevice, st));
      } else {
        h.push_back(rel);
      }
      pre(r.p, z.p);
      const double rz_next = dot(r.p, z.p), beta = rz_next / rz, one = 1.0;
      SGW_BLAS(cublasDscal(blas, m, &beta, p.p, 1));  // p = z + beta p
      SGW_BLAS(cublasDaxpy(blas, m, &one, z.p, 1, p.p, 1));
      rz = rz_next;
    }
  }
  SGW_CUDA(cudaStreamSynchronize(st));
  if (hist) *hist = std::move(h);
  return it;
}

}  // namespace sgw
