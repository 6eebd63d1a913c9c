// PCG hot path: batched packed-symmetric SYMV (SchurSystem::matvec, NN2 local
// solves), the NN2 coarse problem and the CG vector algebra, all with fixed-
// order (atomic-free) reductions so runs are bitwise reproducible.
//
// Reference: src/dd.cpp:142-157 (matvec), :199-253 (apply_nn2), src/pcg.cpp:7-50.
#include <cmath>

#include <set>

#include "solver.cuh"
#include "tiles.cuh"

namespace sgw {

std::atomic<long long> g_launches{0};

enum Scal { RZ = 0, RZN = 1, PQ = 2, RR = 3, BB = 4, RT = 5, TMP = 6, NSCAL = 8 };
constexpr int kRedBlocks = 512;  // max partial-sum blocks of a reduction

// ------------------------------------------------------------ reductions ---
// Block sum in fixed tree order, then the last block to finish sums the block
// partials in index order: deterministic regardless of scheduling.
__device__ void finalize_sum(double v, double* partials, unsigned* counter, double* out, double* out_prev) {
  __shared__ double sh[32];
  __shared__ bool last;
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    double s = lane < (blockDim.x >> 5) ? sh[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) {
      partials[blockIdx.x] = s;
      __threadfence();
      last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (last && w == 0) {
    __threadfence();
    double s = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) s += ((volatile double*)partials)[b];
    s = warp_sum(s);
    if (lane == 0) {
      if (out_prev) *out_prev = *out;
      *out = s;
      *counter = 0u;
    }
  }
}

inline int red_grid(long long len) { return std::max(1, std::min<int>(kRedBlocks, cdiv(len, 256))); }

// sum_i a_i b_i (w_i): w = the ownership mask of a sharded interface vector
__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b, const double* __restrict__ w,
                           long long n, double* partials, unsigned* counter, double* out, double* out_prev) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += w ? a[i] * b[i] * w[i] : a[i] * b[i];
  finalize_sum(s, partials, counter, out, out_prev);
}

// x += alpha p ; r -= alpha q ; rr = r.r   with alpha = scal[RZN] / scal[PQ]
__global__ void cg_xr_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                             const double* __restrict__ q, const double* __restrict__ w, long long n, double* scal,
                             double* partials, unsigned* counter) {
  const double alpha = scal[RZN] / scal[PQ];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    s += w ? ri * ri * w[i] : ri * ri;
  }
  finalize_sum(s, partials, counter, scal + RR, nullptr);
}

// p = z + (rz_next / rz) p  (src/pcg.cpp:45-47); first == 1: p = z
__global__ void cg_p_kernel(double* __restrict__ p, const double* __restrict__ z, long long n, const double* scal,
                            int first) {
  const double beta = first ? 0.0 : scal[RZN] / scal[RZ];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = first ? z[i] : z[i] + beta * p[i];
}

// rt = b - ax ; scal[RT] = rt.rt
__global__ void residual_kernel(double* __restrict__ rt, const double* __restrict__ b, const double* __restrict__ ax,
                                const double* __restrict__ w, long long n, double* scal, double* partials,
                                unsigned* counter) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = b[i] - ax[i];
    rt[i] = v;
    s += w ? v * v * w[i] : v * v;
  }
  finalize_sum(s, partials, counter, scal + RT, nullptr);
}

// (I (x) M) x = b by CG (initial acceleration, src/sg.cpp:370-376).  M is
// SPD with kappa < 10, so CG reaches 1e-16 relative in a few dozen
// iterations.  The scalars stay on the device (the interface CG's kernels with
// z = r); the host reads r.r every 4 iterations only.
void GpuSolver::mass_solve(double* x, const double* b) {
  const long long N = (long long)NSTATE;
  if (mass_w_.n != 3 * (size_t)N) mass_w_.alloc(3 * (size_t)N);
  double *r = mass_w_.p, *p = mass_w_.p + N, *q = mass_w_.p + 2 * N;
  SGW_CUDA(cudaMemsetAsync(x, 0, N * sizeof(double), st_));
  SGW_CUDA(cudaMemcpyAsync(r, b, N * sizeof(double), cudaMemcpyDeviceToDevice, st_));
  SGW_CUDA(cudaMemcpyAsync(p, b, N * sizeof(double), cudaMemcpyDeviceToDevice, st_));
  const double bb = dot_host(b, b, N, false);
  if (bb == 0.0) return;
  const int grid = red_grid(N);
  dot_kernel<<<grid, 256, 0, st_>>>(r, r, nullptr, N, dpart.p, dcount.p, scal.p + RZN, nullptr);  // rz = r.r
  SGW_LAUNCHED();
  for (int it = 0; it < 500;) {
    for (int u = 0; u < 4; ++u, ++it) {
      apply_block(0, p, q);
      dot_kernel<<<grid, 256, 0, st_>>>(p, q, nullptr, N, dpart.p, dcount.p, scal.p + PQ, nullptr);
      SGW_LAUNCHED();
      cg_xr_kernel<<<grid, 256, 0, st_>>>(x, r, p, q, nullptr, N, scal.p, dpart.p, dcount.p);  // alpha = rz / pq
      SGW_LAUNCHED();
      dot_kernel<<<grid, 256, 0, st_>>>(r, r, nullptr, N, dpart.p, dcount.p, scal.p + RZN, scal.p + RZ);
      SGW_LAUNCHED();
      cg_p_kernel<<<grid, 256, 0, st_>>>(p, r, N, scal.p, 0);  // p = r + (rz_new / rz) p
      SGW_LAUNCHED();
    }
    double rr = 0.0;
    SGW_CUDA(cudaMemcpyAsync(&rr, scal.p + RZN, sizeof(double), cudaMemcpyDeviceToHost, st_));
    SGW_CUDA(cudaStreamSynchronize(st_));
    if (!(rr > 1e-32 * bb)) break;
  }
}

// ------------------------------------------------------------- TilePack ----
void TilePack::plan(const std::vector<int>& dims, bool alloc_tiles) {
  nmat = int(dims.size());
  dim = dims;
  ntile.resize(nmat);
  tile_base.resize(nmat + 1);
  xoff.resize(nmat + 1);
  tile_base[0] = 0;
  xoff[0] = 0;
  std::vector<int4> h;
  std::vector<int2> ht;
  for (int s = 0; s < nmat; ++s) {
    ntile[s] = cdiv(dims[s], kTile);
    tile_base[s + 1] = tile_base[s] + (long long)ntile[s] * (ntile[s] + 1) / 2;
    xoff[s + 1] = xoff[s] + (long long)kTile * ntile[s];
    for (int I = 0; I < ntile[s]; ++I)
      for (int J = 0; J <= I; ++J) {
        h.push_back(make_int4(s, I, J, 0));
        ht.push_back(make_int2(int(xoff[s] + (long long)I * kTile), int(xoff[s] + (long long)J * kTile)));
      }
  }
  tx.upload(ht);
  n_tiles = tile_base[nmat];
  xlen = xoff[nmat];
  desc.upload(h);
  if (alloc_tiles) {
    tiles.alloc(size_t(n_tiles) * kTile * kTile);
    rowpart.alloc(size_t(n_tiles) * kTile);
    colpart.alloc(size_t(n_tiles) * kTile);
  }
  d_tile_base.upload(tile_base);
  d_xoff.upload(xoff);
  d_ntile.upload(ntile);
  d_dim.upload(dim);
}

// Pack dense symmetric matrix s (column-major, leading dim ld, lower triangle
// authoritative) into its lower tiles.  One CTA per tile.
__global__ void pack_tiles_kernel(const int4* __restrict__ desc, int n, double* __restrict__ tiles,
                                  const double* __restrict__ A, int L) {
  const long long t = blockIdx.x;
  const int4 d = desc[t];
  const int I = d.y, J = d.z;
  for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
    const int r = e / kTile, c = e % kTile, R = I * kTile + r, Cc = J * kTile + c;
    double v = 0.0;
    if (R < n && Cc < n) v = R >= Cc ? A[(size_t)Cc * L + R] : A[(size_t)R * L + Cc];
    tiles[t * kTile * kTile + e] = v;
  }
}

void pack_tiles_range(TilePack& tp, int s, const double* src, int ld, cudaStream_t st) {
  const long long tb = tp.tile_base[s], te = tp.tile_base[s + 1];
  if (te <= tb) return;
  pack_tiles_kernel<<<(unsigned)(te - tb), 256, 0, st>>>(tp.desc.p + tb, tp.dim[s], tp.tiles.p + tb * kTile * kTile,
                                                         src, ld);
  SGW_LAUNCHED();
}

// Inverse of pack_tiles_kernel: lower tiles of matrix s -> dense column-major
// n x n (both triangles).  One CTA per tile.
__global__ void unpack_tiles_kernel(const int4* __restrict__ desc, int n, const double* __restrict__ tiles,
                                    double* __restrict__ A) {
  const long long t = blockIdx.x;
  const int4 d = desc[t];
  for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
    const int r = e / kTile, c = e % kTile, R = d.y * kTile + r, Cc = d.z * kTile + c;
    if (R >= n || Cc >= n || Cc > R) continue;
    const double v = tiles[t * kTile * kTile + e];
    A[(size_t)Cc * n + R] = v;
    A[(size_t)R * n + Cc] = v;
  }
}

// Dense copy of subdomain s's local operator (verification hook): which 0 =
// S_s (a x a), 1 = Q_s = S_rr^-1 (r x r), 2 = Psi_s (r x c), column-major.
std::vector<double> GpuSolver::local_block(int s, int which, std::vector<long long>* gmap) {
  if (s < 0 || s >= NS) throw Error(1, "local_block: subdomain not on this rank");
  std::vector<double> out;
  const int a = NT * ng_[s], r = NT * nr_[s], c = NT * nc_[s];
  if (which == 0 || which == 1) {
    TilePack& tp = which == 0 ? Sp : Qp;
    if (!tp.tiles.p) throw Error(1, "local_block: S tiles are not stored (reduced-memory mode)");
    const int dim = which == 0 ? a : r;
    DBuf<double> d;
    d.alloc(std::max<size_t>(1, (size_t)dim * dim));
    const long long tb = tp.tile_base[s], te = tp.tile_base[s + 1];
    if (te > tb) {
      unpack_tiles_kernel<<<(unsigned)(te - tb), 256, 0, st_>>>(tp.desc.p + tb, dim, tp.tiles.p + tb * kTile * kTile,
                                                               d.p);
      SGW_LAUNCHED();
    }
    out.resize((size_t)dim * dim);
    SGW_CUDA(cudaMemcpyAsync(out.data(), d.p, out.size() * sizeof(double), cudaMemcpyDeviceToHost, st_));
  } else if (which == 2) {
    out.resize((size_t)r * c);
    if (!out.empty())
      SGW_CUDA(cudaMemcpyAsync(out.data(), Psi.p + psioff_[s], out.size() * sizeof(double), cudaMemcpyDeviceToHost,
                               st_));
  } else {
    throw Error(1, "local_block: which must be 0 (S), 1 (S_rr^-1) or 2 (Psi)");
  }
  SGW_CUDA(cudaStreamSynchronize(st_));
  if (gmap) {  // flat local index j*ng + p -> global flat interface index (make_flat_maps, dd.cpp:78-96)
    const auto& sd = G.sub[s];
    gmap->resize(a);
    for (int j = 0; j < NT; ++j)
      for (int p = 0; p < ng_[s]; ++p)
        (*gmap)[(size_t)j * ng_[s] + p] = (long long)j * G.n_iface_global + G.iface_gpos[sd.iface_pos[p]];
  }
  return out;
}

// One CTA (8 warps) per 64x64 lower tile (tiles.cuh): row / column partials.
__global__ void __launch_bounds__(256) symv_tiles_kernel(const int4* __restrict__ desc,
                                                         const double* __restrict__ tiles,
                                                         const long long* __restrict__ xoff,
                                                         const double* __restrict__ x,
                                                         double* __restrict__ rowpart,
                                                         double* __restrict__ colpart) {
  __shared__ double csum[8][kTile];
  const long long t = blockIdx.x;
  const int4 d = desc[t];
  const double* xb = x + xoff[d.x];
  tile_symv(tiles + t * (kTile * kTile), xb + d.y * kTile, xb + d.z * kTile, d.y == d.z, rowpart + t * kTile,
            colpart + t * kTile, csum);
}


void GpuSolver::symv(TilePack& tp, const double* xloc, double*) {
  if (!tp.n_tiles) return;
  cudaEvent_t e0;
  KP.begin(&tp == &Sp ? K_SYMV_S : K_SYMV_Q, st_, &e0);
  symv_tiles_kernel<<<(unsigned)tp.n_tiles, 256, 0, st_>>>(tp.desc.p, tp.tiles.p, tp.d_xoff.p, xloc, tp.rowpart.p,
                                                          tp.colpart.p);
  SGW_LAUNCHED();
  KP.end(st_);
}

static double packed_bytes(const std::vector<int>& dims) {
  double b = 0;
  for (int a : dims) b += 0.5 * double(a) * (a + 1) * 8.0;
  return b;
}
double GpuSolver::bytes_S() const { return packed_bytes(Sp.dim); }
double GpuSolver::bytes_Q() const { return packed_bytes(Qp.dim); }
// B_iter = 8 [sum_s (a(a+1)/2 + r(r+1)/2 + 2 r c) + n_C (n_C+1)/2 + 12 (P+1) n_G]
double GpuSolver::bytes_iter() const {
  double b = bytes_S() + bytes_Q();
  for (int s = 0; s < NS; ++s) b += 2.0 * 8.0 * double(NT * nr_[s]) * double(NT * nc_[s]);
  b += 8.0 * 0.5 * double(NC) * (NC + 1);
  b += 8.0 * 12.0 * NG;
  return b;
}
double GpuSolver::bytes_sgop() const {
  // JIT operator: 2 stored couplings per node and input term (sgop.cu), x read
  // and y written once: 8 n [2 n_in + 2 (P+1)].  Table-driven kernel: the
  // SURVEY 8d 3-value stored form 8 n [3 n_in + 2 (P+1)].
  return 8.0 * n * ((sgop_ ? 2.0 : 3.0) * NIN + 2.0 * NT);
}
double GpuSolver::flops_sgop() const {
  if (sgop_) return sgop_flops(*sgop_, n);
  // SURVEY 8d F_op = 2 n [5 N_ij + nnzG_full + 7 (P+1)] (5-point stencils)
  std::set<std::pair<int, int>> ij;
  long long full = 0;
  for (size_t e = 0; e < P.tensor.v.size(); ++e) {
    ij.insert({P.tensor.i[e], P.tensor.j[e]}), ij.insert({P.tensor.i[e], P.tensor.k[e]});
    full += P.tensor.j[e] == P.tensor.k[e] ? 1 : 2;
  }
  return 2.0 * n * (5.0 * double(ij.size()) + double(full) + 7.0 * NT);
}

// ---------------------------------------------------- gather / scatter -----
// LI[s][j*ng+p] = (w) X[j*n_iface + iface_pos[s][p]]
__global__ void gather_li_kernel(const double* __restrict__ X, double* __restrict__ li, const long long* __restrict__ xoff,
                                 const int* __restrict__ ip_off, const int* __restrict__ iface_pos,
                                 const double* __restrict__ w, const int* __restrict__ ng, int ns, int nt,
                                 int n_iface, int weighted) {
  const int s = blockIdx.y;
  const int a = ng[s] * nt;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < a; f += gridDim.x * blockDim.x) {
    const int j = f / ng[s], p = f % ng[s];
    double v = X[(long long)j * n_iface + iface_pos[ip_off[s] + p]];
    if (weighted) v *= w[ip_off[s] + p];
    li[xoff[s] + f] = v;
  }
}

void GpuSolver::gather_li(const double* glob, double* li, bool weighted) {
  dim3 grid(cdiv(NT * 4 * (G.mx + G.my), 256), NS);
  gather_li_kernel<<<grid, 256, 0, st_>>>(glob, li, Sp.d_xoff.p, ip_off.p, iface_pos.p, iface_w.p, ng_d.p, NS, NT,
                                           G.n_iface, weighted ? 1 : 0);
  SGW_LAUNCHED();
}

// X[q] = sum over subdomains sharing interface node q (ascending s) of
//        (w) * (tiles ? tile_reduce(S) : LI)[s][j*ng+p]   ;  optional dot(X, dw)
template <bool FromTiles>
__global__ void scatter_kernel(double* __restrict__ X, const double* __restrict__ li, const long long* __restrict__ xoff,
                               const int* __restrict__ ip_off, const double* __restrict__ w,
                               const int* __restrict__ inv_cnt, const int* __restrict__ inv_s,
                               const int* __restrict__ inv_p, const int* __restrict__ ng, int n_iface, long long NG,
                               int weighted, const double* __restrict__ rowpart, const double* __restrict__ colpart,
                               const long long* __restrict__ tile_base, const int* __restrict__ ntile,
                               const double* __restrict__ dw, double* partials, unsigned* counter, double* dout) {
  double acc = 0.0;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < NG; q += (long long)gridDim.x * blockDim.x) {
    const int j = int(q / n_iface), g = int(q % n_iface);
    double y = 0.0;
    for (int e = 0; e < inv_cnt[g]; ++e) {
      const int s = inv_s[4 * g + e], p = inv_p[4 * g + e];
      const int f = j * ng[s] + p;
      double v = FromTiles ? tile_reduce(rowpart, colpart, tile_base[s], ntile[s], f) : li[xoff[s] + f];
      if (weighted) v *= w[ip_off[s] + p];
      y += v;
    }
    X[q] = y;
    if (dw) acc += y * dw[q];
  }
  if (dw) finalize_sum(acc, partials, counter, dout, nullptr);
}

// scatter_kernel<true> on the CTA partials of a tile walk (walk_kernel)
__global__ void scatter_range_kernel(double* __restrict__ X, const RangePack P, const int* __restrict__ inv_cnt,
                                     const int* __restrict__ inv_s, const int* __restrict__ inv_p,
                                     const int* __restrict__ ng, int n_iface, long long NG,
                                     const double* __restrict__ dw, double* partials, unsigned* counter,
                                     double* dout) {
  double acc = 0.0;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < NG; q += (long long)gridDim.x * blockDim.x) {
    const int j = int(q / n_iface), g = int(q % n_iface);
    double y = 0.0;
    for (int e = 0; e < inv_cnt[g]; ++e) {
      const int s = inv_s[4 * g + e], p = inv_p[4 * g + e];
      y += range_reduce(P, s, j * ng[s] + p);
    }
    X[q] = y;
    if (dw) acc += y * dw[q];
  }
  if (dw) finalize_sum(acc, partials, counter, dout, nullptr);
}

// S x (no exchange): the stored S tiles, by a tile walk when the ranges exist
void GpuSolver::s_product(const double* x, double* y, const double* dot_with, double* dot_out) {
  const int grid = red_grid(NG);
  gather_li(x, li_x.p, false);
  if (walk_ok_) {
    walk_pack(0, li_x.p);
    scatter_range_kernel<<<grid, 256, 0, st_>>>(y, range_pack(0), inv_cnt.p, inv_s.p, inv_p.p, ng_d.p, G.n_iface, NG,
                                                dot_with, dpart.p, dcount.p, dot_out);
  } else {
    symv(Sp, li_x.p, nullptr);
    scatter_kernel<true><<<grid, 256, 0, st_>>>(y, nullptr, Sp.d_xoff.p, ip_off.p, iface_w.p, inv_cnt.p, inv_s.p,
                                                inv_p.p, ng_d.p, G.n_iface, NG, 0, Sp.rowpart.p, Sp.colpart.p,
                                                Sp.d_tile_base.p, Sp.d_ntile.p, dot_with, dpart.p, dcount.p, dot_out);
  }
  SGW_LAUNCHED();
}

void GpuSolver::scatter_li(const double* li, double* glob, bool weighted, double* dot_with, double* dot_out) {
  const int grid = red_grid(NG);
  scatter_kernel<false><<<grid, 256, 0, st_>>>(glob, li, Sp.d_xoff.p, ip_off.p, iface_w.p, inv_cnt.p, inv_s.p,
                                               inv_p.p, ng_d.p, G.n_iface, NG, weighted ? 1 : 0, nullptr, nullptr,
                                               nullptr, nullptr, dot_with, dpart.p, dcount.p, dot_out);
  SGW_LAUNCHED();
}

// --------------------------------------------------------------- matvec ----
void GpuSolver::schur_matvec(const double* x, double* y) {
  if (P.implicit_schur) return schur_matvec_implicit(x, y);
  s_product(x, y, nullptr, nullptr);
  halo_sum(y);  // sharded: partial sums over owned subdomains -> full sums
  ++T.matvecs;
}

// ------------------------------------------------------------------ NN2 ----
// f = D_s R_s r split into f_r (r-space, padded per subdomain) and f_c.
__global__ void nn2_gather_kernel(const double* __restrict__ r, const int* __restrict__ r_gidx,
                                  const double* __restrict__ r_w, double* __restrict__ fr, long long nr_tot,
                                  const int* __restrict__ c_gidx, const double* __restrict__ c_w,
                                  double* __restrict__ fc, long long nc_tot) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nr_tot + nc_tot;
       i += (long long)gridDim.x * blockDim.x) {
    if (i < nr_tot) {
      const int gi = r_gidx[i];
      fr[i] = gi >= 0 ? r_w[i] * r[gi] : 0.0;
    } else {
      const long long k = i - nr_tot;
      const int gi = c_gidx[k];
      fc[k] = gi >= 0 ? c_w[k] * r[gi] : 0.0;
    }
  }
}

// d_s = f_c - Psi^T f_r   (= f_c - S_rc^T S_rr^-1 f_r, src/dd.cpp:214-217); warp per (s, c)
__global__ void psi_t_kernel(const double* __restrict__ Psi, const long long* __restrict__ psioff,
                             const double* __restrict__ fr, const long long* __restrict__ roff,
                             const double* __restrict__ fc, const long long* __restrict__ coff,
                             double* __restrict__ dsub, const int* __restrict__ nr, const int* __restrict__ nc,
                             int nt, int ns) {
  const int s = blockIdx.y;
  const int csz = nc[s] * nt, rsz = nr[s] * nt;
  const int lane = threadIdx.x & 31;
  for (int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < csz; c += gridDim.x * (blockDim.x >> 5)) {
    const double* col = Psi + psioff[s] + (long long)c * rsz;
    const double* f = fr + roff[s];
    double acc = 0.0;
    for (int a = lane; a < rsz; a += 32) acc += col[a] * f[a];
    acc = warp_sum(acc);
    if (lane == 0) dsub[coff[s] + c] = fc[coff[s] + c] - acc;
  }
}

// d = sum_s B_s^T d_s in ascending s (src/dd.cpp:221-226)
__global__ void coarse_assemble_kernel(const double* __restrict__ dsub, const long long* __restrict__ coff,
                                       const int* __restrict__ cinv_cnt, const int* __restrict__ cinv_s,
                                       const int* __restrict__ cinv_c, const int* __restrict__ nc, int n_corner,
                                       int NC, double* __restrict__ d) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < NC; q += gridDim.x * blockDim.x) {
    const int j = q / n_corner, g = q % n_corner;
    double acc = 0.0;
    for (int e = 0; e < cinv_cnt[g]; ++e) {
      const int s = cinv_s[4 * g + e];
      acc += dsub[coff[s] + j * nc[s] + cinv_c[4 * g + e]];
    }
    d[q] = acc;
  }
}

// y = A x for a symmetric column-major n x n A (warp per row = column)
__global__ void symv_dense_kernel(const double* __restrict__ A, const double* __restrict__ x, double* __restrict__ y,
                                  int n) {
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += gridDim.x * (blockDim.x >> 5)) {
    const double* col = A + (long long)r * n;
    double acc = 0.0;
    for (int c = lane; c < n; c += 32) acc += col[c] * x[c];
    acc = warp_sum(acc);
    if (lane == 0) y[r] = acc;
  }
}

// zeta_s on the local interface: remaining  u_r = Q f_r - Psi u_c(s)  (tile partials of Q),
// corners u_c(s)  (src/dd.cpp:230-246).  Unweighted; the scatter applies D_s.
__global__ void nn2_local_kernel(double* __restrict__ li, const long long* __restrict__ lioff,
                                 const int* __restrict__ ip_off, const int* __restrict__ pkind,
                                 const int* __restrict__ ng, const int* __restrict__ nr, const int* __restrict__ nc,
                                 int nt, const double* __restrict__ rowpart, const double* __restrict__ colpart,
                                 const long long* __restrict__ qbase, const int* __restrict__ qnt,
                                 const double* __restrict__ Psi, const long long* __restrict__ psioff,
                                 const double* __restrict__ uc, const int* __restrict__ corner_pos_flat,
                                 const int* __restrict__ cp_off, int n_corner, int has_coarse) {
  const int s = blockIdx.y;
  const int a = ng[s] * nt, rsz = nr[s] * nt, ncs = nc[s];
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < a; f += gridDim.x * blockDim.x) {
    const int j = f / ng[s], p = f % ng[s];
    const int k = pkind[ip_off[s] + p];
    double v;
    if (k >= 0) {  // remaining dof: r-space index j*nr + k
      const int ar = j * nr[s] + k;
      v = tile_reduce(rowpart, colpart, qbase[s], qnt[s], ar);
      if (has_coarse) {
        const double* P = Psi + psioff[s] + ar;
        for (int jc = 0; jc < nt; ++jc)
          for (int cc = 0; cc < ncs; ++cc)
            v -= P[(long long)(jc * ncs + cc) * rsz] * uc[jc * n_corner + corner_pos_flat[cp_off[s] + cc]];
      }
    } else {
      const int cc = -1 - k;
      v = has_coarse ? uc[j * n_corner + corner_pos_flat[cp_off[s] + cc]] : 0.0;
    }
    li[lioff[s] + f] = v;
  }
}

// d_s = f_c - Psi_s^T f_r from the Psi^T walk's corner partials (c-space, padded per subdomain)
__global__ void psi_t_range_kernel(const RangePack Pp, const double* __restrict__ fc, const long long* __restrict__ coff,
                                   const int* __restrict__ ncs, double* __restrict__ dsub, int ns) {
  const int s = blockIdx.y;
  if (s >= ns) return;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncs[s]; c += gridDim.x * blockDim.x)
    dsub[coff[s] + c] = fc[coff[s] + c] - rect_reduce(Pp, s, c);
}
// B_s u_c per subdomain (c-space, compact)
__global__ void ucl_kernel(const double* __restrict__ uc, const long long* __restrict__ coff,
                           const int* __restrict__ nc, const int* __restrict__ corner_pos_flat,
                           const int* __restrict__ cp_off, int nt, int n_corner, double* __restrict__ ucl) {
  const int s = blockIdx.y;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nt * nc[s]; c += gridDim.x * blockDim.x) {
    const int j = c / nc[s], cc = c % nc[s];
    ucl[coff[s] + c] = uc[j * n_corner + corner_pos_flat[cp_off[s] + cc]];
  }
}
// z_s from the Q walk and the second Psi^T walk (remaining-dof part of its partials)
__global__ void nn2_local_walk_kernel(double* __restrict__ li, const long long* __restrict__ lioff,
                                      const int* __restrict__ ip_off, const int* __restrict__ pkind,
                                      const int* __restrict__ ng, const int* __restrict__ nr,
                                      const int* __restrict__ nc, int nt, const RangePack Pq, const RangePack Pp,
                                      const double* __restrict__ ucl, const long long* __restrict__ coff,
                                      int has_coarse) {
  const int s = blockIdx.y;
  const int a = ng[s] * nt;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < a; f += gridDim.x * blockDim.x) {
    const int j = f / ng[s], p = f % ng[s];
    const int k = pkind[ip_off[s] + p];
    double v;
    if (k >= 0) {
      const int ar = j * nr[s] + k;
      v = range_reduce(Pq, s, ar);
      if (has_coarse) v -= rect_reduce(Pp, s, kTile * Pp.nI[s] + ar);
    } else {
      v = has_coarse ? ucl[coff[s] + (long long)j * nc[s] + (-1 - k)] : 0.0;
    }
    li[lioff[s] + f] = v;
  }
}

void GpuSolver::apply_nn2(const double* r, double* z) {
  const long long nr_tot = roff_.back(), nc_tot = coff_.back();
  nn2_gather_kernel<<<red_grid(nr_tot + nc_tot), 256, 0, st_>>>(r, r_gidx.p, r_w.p, r_x.p, nr_tot, c_gidx.p, c_w.p,
                                                                 c_f.p, nc_tot);
  SGW_LAUNCHED();
  const bool has_coarse = NC > 0;
  if (walk_ok_) {  // Q, Psi^T f_r, F_cc^-1, Psi u_c as tile walks (pcg_fused.cu)
    walk_pack(1, r_x.p);
    if (has_coarse) {
      walk_psi(1, r_x.p);
      psi_t_range_kernel<<<dim3(cdiv(NT * 4, 128), NS), 128, 0, st_>>>(psi_pack(), c_f.p, d_coff.p, psi_ncs_.p, c_d.p,
                                                                     NS);
      SGW_LAUNCHED();
      coarse_assemble_kernel<<<cdiv(NC, 256), 256, 0, st_>>>(c_d.p, d_coff.p, cinv_cnt.p, cinv_s.p, cinv_c.p, nc_d.p,
                                                             G.n_corner, NC, dcoarse.p);
      SGW_LAUNCHED();
      allreduce(dcoarse.p, NC);
      symv_dense_kernel<<<cdiv(NC, 8), 256, 0, st_>>>(Finv.p, dcoarse.p, ucoarse.p, NC);
      SGW_LAUNCHED();
      ucl_kernel<<<dim3(cdiv(NT * 4, 128), NS), 128, 0, st_>>>(ucoarse.p, d_coff.p, nc_d.p, cpos_flat_.p, cp_off_.p,
                                                             NT, G.n_corner, ucl_.p);
      SGW_LAUNCHED();
      walk_psi(2, ucl_.p);
    }
    nn2_local_walk_kernel<<<dim3(cdiv(NT * 4 * (G.mx + G.my), 256), NS), 256, 0, st_>>>(
        li_y.p, Sp.d_xoff.p, ip_off.p, pkind_.p, ng_d.p, nr_d.p, nc_d.p, NT, range_pack(1), psi_pack(), ucl_.p,
        d_coff.p, has_coarse ? 1 : 0);
    SGW_LAUNCHED();
    scatter_li(li_y.p, z, true, nullptr, nullptr);
    halo_sum(z);
    ++T.nn2s;
    return;
  }
  symv(Qp, r_x.p, nullptr);
  if (has_coarse) {
    psi_t_kernel<<<dim3(cdiv(NT * 4, 8), NS), 256, 0, st_>>>(Psi.p, d_psioff.p, r_x.p, d_roff.p, c_f.p, d_coff.p,
                                                              c_d.p, nr_d.p, nc_d.p, NT, NS);
    SGW_LAUNCHED();
    coarse_assemble_kernel<<<cdiv(NC, 256), 256, 0, st_>>>(c_d.p, d_coff.p, cinv_cnt.p, cinv_s.p, cinv_c.p, nc_d.p,
                                                           G.n_corner, NC, dcoarse.p);
    SGW_LAUNCHED();
    allreduce(dcoarse.p, NC);
    symv_dense_kernel<<<cdiv(NC, 8), 256, 0, st_>>>(Finv.p, dcoarse.p, ucoarse.p, NC);
    SGW_LAUNCHED();
  }
  nn2_local_kernel<<<dim3(cdiv(NT * 4 * (G.mx + G.my), 256), NS), 256, 0, st_>>>(
        li_y.p, Sp.d_xoff.p, ip_off.p, pkind_.p, ng_d.p, nr_d.p, nc_d.p, NT, Qp.rowpart.p, Qp.colpart.p,
        Qp.d_tile_base.p, Qp.d_ntile.p, Psi.p, d_psioff.p, ucoarse.p, cpos_flat_.p, cp_off_.p, G.n_corner,
        has_coarse ? 1 : 0);
  SGW_LAUNCHED();
  scatter_li(li_y.p, z, true, nullptr, nullptr);
  halo_sum(z);
  ++T.nn2s;
}

// ------------------------------------------------------- lumped / NN1 ----
// z = sum_s R_s^T D_s A_s D_s R_s r (dd.cpp:159-195), A_s = S_s^-1 (NN1) or
// K~_GG,s (lumped), both held as packed symmetric tiles
void GpuSolver::apply_one_level(TilePack& tp, const double* r, double* z) {
  gather_li(r, li_x.p, true);
  symv(tp, li_x.p, nullptr);
  const int grid = red_grid(NG);
  scatter_kernel<true><<<grid, 256, 0, st_>>>(z, nullptr, tp.d_xoff.p, ip_off.p, iface_w.p, inv_cnt.p, inv_s.p,
                                              inv_p.p, ng_d.p, G.n_iface, NG, 1, tp.rowpart.p, tp.colpart.p,
                                              tp.d_tile_base.p, tp.d_ntile.p, nullptr, nullptr, nullptr, nullptr);
  SGW_LAUNCHED();
  halo_sum(z);
  ++T.nn2s;
}

void GpuSolver::apply_precond(int kind, const double* r, double* z) {
  if (kind == 0) return apply_nn2(r, z);
  TilePack& tp = kind == 1 ? Sinvp : Aggp;
  if (kind < 0 || kind > 2 || tp.nmat == 0)
    throw Error(1, "preconditioner not built: construct the solver with this preconditioner");
  apply_one_level(tp, r, z);
}

// -------------------------------------------------------------- vectors ----
// iface: a, b are (sharded) interface vectors: owned entries only, summed over ranks
void GpuSolver::dot_dev(const double* a, const double* b, long long len, double* out, bool iface) {
  dot_kernel<<<red_grid(len), 256, 0, st_>>>(a, b, iface ? dot_mask() : nullptr, len, dpart.p, dcount.p, out, nullptr);
  SGW_LAUNCHED();
  if (iface) allreduce(out, 1);
}

double GpuSolver::dot_host(const double* a, const double* b, long long len, bool iface) {
  dot_dev(a, b, len, scal.p + TMP, iface);
  double h = 0;
  SGW_CUDA(cudaMemcpyAsync(&h, scal.p + TMP, sizeof(double), cudaMemcpyDeviceToHost, st_));
  SGW_CUDA(cudaStreamSynchronize(st_));
  return h;
}

// ------------------------------------------------------------------ PCG ----
// src/pcg.cpp:7-50: x0 = 0; stop on the recurrence residual, confirm with the
// true residual, restart from it (without resetting p) if the check fails.
int GpuSolver::pcg(const double* b, double* x, bool* converged, std::vector<double>* hist) {
  if (fused_ok()) return pcg_fused(b, x, converged, hist);
  if (phase_ok()) return pcg_phase(b, x, converged, hist);
  cudaEventRecord(ev_[0], st_);
  const long long N = NG;
  const int grid = red_grid(N);
  SGW_CUDA(cudaMemsetAsync(x, 0, N * sizeof(double), st_));
  const double bb = dot_host(b, b, N, true);
  const double bnorm = std::sqrt(bb);
  int iters = 0;
  *converged = false;
  if (hist) hist->clear();
  if (bnorm == 0.0) {
    *converged = true;
    last_rel = 0.0;
    if (hist) hist->push_back(0.0);
    cudaEventRecord(ev_[1], st_);
    cudaEventSynchronize(ev_[1]);
    float ms = 0;
    cudaEventElapsedTime(&ms, ev_[0], ev_[1]);
    T.pcg_ms += ms;
    return 0;
  }
  const double* w = dot_mask();  // sharded: owned interface entries (global dots)
  // r.z -> scal[RZN] (previous in scal[RZ]), summed over ranks
  auto rz_dot = [&]() {
    dot_kernel<<<grid, 256, 0, st_>>>(vr.p, vz.p, w, N, dpart.p, dcount.p, scal.p + RZN, scal.p + RZ);
    SGW_LAUNCHED();
    allreduce(scal.p + RZN, 1);
  };
  SGW_CUDA(cudaMemcpyAsync(vr.p, b, N * sizeof(double), cudaMemcpyDeviceToDevice, st_));
  apply_precond(P.precond, vr.p, vz.p);
  rz_dot();
  cg_p_kernel<<<grid, 256, 0, st_>>>(vp.p, vz.p, N, scal.p, 1);
  SGW_LAUNCHED();
  if (hist) hist->push_back(1.0);
  // The two halves of an iteration (S p ... x, r, ||r||; NN2 ... p) as CUDA
  // graphs when the exchange can be captured (no exchange, or NCCL): two
  // launches per iteration instead of ~15 kernels and the collectives.
  const bool graphs = !comm_ || comm_->capturable();
  auto matvec_half = [&]() {
    if (P.implicit_schur) {
      schur_matvec_implicit(vp.p, vq.p);  // halo included
      dot_kernel<<<grid, 256, 0, st_>>>(vp.p, vq.p, w, N, dpart.p, dcount.p, scal.p + PQ, nullptr);
      SGW_LAUNCHED();
    } else if (!comm_) {
      s_product(vp.p, vq.p, vp.p, scal.p + PQ);  // p.q fused into the scatter
    } else {
      s_product(vp.p, vq.p, nullptr, nullptr);
      halo_sum(vq.p);
      dot_kernel<<<grid, 256, 0, st_>>>(vp.p, vq.p, w, N, dpart.p, dcount.p, scal.p + PQ, nullptr);
      SGW_LAUNCHED();
    }
    allreduce(scal.p + PQ, 1);
    cg_xr_kernel<<<grid, 256, 0, st_>>>(x, vr.p, vp.p, vq.p, w, N, scal.p, dpart.p, dcount.p);
    SGW_LAUNCHED();
    allreduce(scal.p + RR, 1);
    SGW_CUDA(cudaMemcpyAsync(h_scal_, scal.p + RR, sizeof(double), cudaMemcpyDeviceToHost, st_));
  };
  auto precond_half = [&]() {
    apply_precond(P.precond, vr.p, vz.p);
    rz_dot();
    cg_p_kernel<<<grid, 256, 0, st_>>>(vp.p, vz.p, N, scal.p, 0);
    SGW_LAUNCHED();
  };
  if (graphs && (graph_x_ != x || !graph_mv_)) {
    for (cudaGraphExec_t* ge : {&graph_mv_, &graph_pc_})
      if (*ge) cudaGraphExecDestroy(*ge), *ge = nullptr;
    long long* cnt[2] = {&graph_mv_launches_, &graph_pc_launches_};
    cudaGraphExec_t* ex[2] = {&graph_mv_, &graph_pc_};
    const bool kp = KP.on;
    KP.on = false;  // no per-kernel events inside the graphs (PCG time is still timed)
    for (int h = 0; h < 2; ++h) {
      const long long l0 = g_launches.load();
      cudaGraph_t gr;
      SGW_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeRelaxed));
      if (h == 0) matvec_half(); else precond_half();
      SGW_CUDA(cudaStreamEndCapture(st_, &gr));
      SGW_CUDA(cudaGraphInstantiate(ex[h], gr, 0));
      cudaGraphDestroy(gr);
      *cnt[h] = g_launches.load() - l0;
      g_launches -= *cnt[h];  // counted per replay below
    }
    KP.on = kp;
    graph_x_ = x;
  }
  for (int it = 0; it < P.max_iter; ++it) {
    // q = S p, p.q, x, r, ||r||^2 -> host
    if (graphs) {
      SGW_CUDA(cudaGraphLaunch(graph_mv_, st_));
      g_launches += graph_mv_launches_;
    } else {
      matvec_half();
    }
    ++T.matvecs;
    ++iters;
    SGW_CUDA(cudaStreamSynchronize(st_));
    if (comm_) comm_->poll();
    double rel = std::sqrt(*h_scal_) / bnorm;
    last_rel = rel;
    if (rel <= P.tol) {
      schur_matvec(x, vq.p);
      residual_kernel<<<grid, 256, 0, st_>>>(vrt.p, b, vq.p, w, N, scal.p, dpart.p, dcount.p);
      SGW_LAUNCHED();
      allreduce(scal.p + RT, 1);
      double rt = 0;
      SGW_CUDA(cudaMemcpyAsync(&rt, scal.p + RT, sizeof(double), cudaMemcpyDeviceToHost, st_));
      SGW_CUDA(cudaStreamSynchronize(st_));
      rel = std::sqrt(rt) / bnorm;
      last_rel = rel;
      if (hist) hist->push_back(rel);
      if (rel <= P.tol) {
        *converged = true;
        break;
      }
      SGW_CUDA(cudaMemcpyAsync(vr.p, vrt.p, N * sizeof(double), cudaMemcpyDeviceToDevice, st_));
    } else if (hist) {
      hist->push_back(rel);
    }
    if (graphs) {
      SGW_CUDA(cudaGraphLaunch(graph_pc_, st_));
      g_launches += graph_pc_launches_;
    } else {
      precond_half();
    }
    T.nn2s += 1;
  }
  cudaEventRecord(ev_[1], st_);
  SGW_CUDA(cudaEventSynchronize(ev_[1]));
  float ms = 0;
  cudaEventElapsedTime(&ms, ev_[0], ev_[1]);
  T.pcg_ms += ms;
  T.iterations += iters;
  return iters;
}

}  // namespace sgw
