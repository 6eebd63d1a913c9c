// Per-Newmark-step kernels: stochastic-Galerkin stencil operator applies
// (global apply_block_*, local force, A_GI / A_IG couplings), the batched
// and the fused Newmark predictor/update (the Dirichlet sweeps are in sweep.cu).
//
// Reference: src/sg.cpp:252-356 (local_force, step_rhs_and_solve),
// src/sg.cpp:358-423 (run), src/sg.cpp:425-447 (apply_block_*),
// src/newmark.cpp:16-49.
#include <cmath>
#include <cstdlib>

#include <cstring>

#include "solver.cuh"

namespace sgw {

__constant__ int sDI[7] = {0, 1, -1, 0, 0, 1, -1};
__constant__ int sDJ[7] = {0, 0, 0, 1, -1, 1, -1};

// coefficient of direction dir from a 3-component (K) or 4-component (M)
// stencil with component stride cs; own node o, neighbour nb.
__device__ __forceinline__ double kco(const double* K, long long cs, long long o, long long nb, int dir) {
  switch (dir) {
    case 0: return __ldg(K + o);
    case 1: return __ldg(K + cs + o);
    case 2: return __ldg(K + cs + nb);
    case 3: return __ldg(K + 2 * cs + o);
    case 4: return __ldg(K + 2 * cs + nb);
    default: return 0.0;
  }
}
__device__ __forceinline__ double mco(const double* M, long long cs, long long o, long long nb, int dir) {
  switch (dir) {
    case 0: return __ldg(M + o);
    case 1: return __ldg(M + cs + o);
    case 2: return __ldg(M + cs + nb);
    case 3: return __ldg(M + 2 * cs + o);
    case 4: return __ldg(M + 2 * cs + nb);
    case 5: return __ldg(M + 3 * cs + o);
    default: return __ldg(M + 3 * cs + nb);
  }
}


// ------------------------------------------------------ global operator ---
// y_k = cm * sum_nb M x_k + ck * sum_{(i,j,g) in G_k} g sum_nb K_i x_j on the
// reduced (nx-1) x (ny-1) dof grid (src/sg.cpp:425-447).  Thread per (d, k).
__global__ void sg_apply_global_kernel(const double* __restrict__ Kg, const double* __restrict__ Mg, int n, int rw,
                                       int rh, int nt, GList g, const double* __restrict__ x, double* __restrict__ y,
                                       double cm, double ck) {
  const long long total = (long long)n * nt;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int d = int(t % n), k = int(t / n);
    const int il = d % rw, jl = d / rw;
    int nb[7];
    bool ok[7];
#pragma unroll
    for (int dir = 0; dir < 7; ++dir) {
      const int i2 = il + sDI[dir], j2 = jl + sDJ[dir];
      ok[dir] = i2 >= 0 && i2 < rw && j2 >= 0 && j2 < rh;
      nb[dir] = ok[dir] ? j2 * rw + i2 : d;
    }
    double ym = 0.0, yk = 0.0;
    if (cm != 0.0) {
      const double* xk = x + (long long)k * n;
#pragma unroll
      for (int dir = 0; dir < 7; ++dir)
        if (ok[dir]) ym += mco(Mg, n, d, nb[dir], dir) * xk[nb[dir]];
    }
    if (ck != 0.0) {
      for (int e = g.ptr[k]; e < g.ptr[k + 1]; ++e) {
        const double* Ki = Kg + (long long)g.i[e] * 3 * n;
        const double* xj = x + (long long)g.j[e] * n;
        double s = 0.0;
#pragma unroll
        for (int dir = 0; dir < 5; ++dir)
          if (ok[dir]) s += kco(Ki, n, d, nb[dir], dir) * xj[nb[dir]];
        yk += g.v[e] * s;
      }
    }
    y[t] = cm * ym + ck * yk;
  }
}

// op 0 (mass only, the initial-acceleration CG) reads no K: the simple kernel;
// ops 1 / 2 stream every K_i: the JIT-specialised fused operator (sgop.cu).
void GpuSolver::apply_block(int op, const double* x, double* y) {
  const double cm = op == 0 ? 1.0 : op == 1 ? 0.0 : P.mass_scale;
  const double ck = op == 0 ? 0.0 : op == 1 ? 1.0 : P.stiff_scale;
  cudaEvent_t e0;
  KP.begin(K_SGOP, st_, &e0);
  if (op == 0 || !sgop_) {
    const long long total = (long long)NSTATE;
    sg_apply_global_kernel<<<std::min(cdiv(total, 256), 8 * kNumSMs * 16), 256, 0, st_>>>(
        Kg.p, Mg.p, n, P.nx - 1, P.ny - 1, NT, GList{gk_ptr.p, gk_i.p, gk_j.p, gk_v.p}, x, y, cm, ck);
    SGW_LAUNCHED();
  } else {
    SgOpArgs a = sgop_args_;
    a.x = x, a.y = y, a.alpha = cm, a.beta = ck;
    launch_sgop(*sgop_, a, st_);
  }
  KP.end(st_);
}

// -------------------------------------------------------- local operators --
// reduced dof of local node (il, jl) of subdomain s; callers only ask for
// non-Dirichlet nodes (lid_to_p != -1)
__device__ __forceinline__ int block_origin(int s, int n, int p) { return (s * n + p - 1) / p; }
__device__ __forceinline__ int lid_dof(const LocalArgs& A, int s, int il, int jl) {
  const int sg = A.sub_gid[s];  // global subdomain id
  const int gi = block_origin(sg % A.px, A.nx, A.px) + il, gj = block_origin(sg / A.px, A.ny, A.py) + jl;
  return (gj - 1) * (A.nx - 1) + gi - 1;
}
__device__ __forceinline__ long long interior_index(const LocalArgs& A, int s, int il, int jl, int term) {
  return ((long long)s * A.H + (jl - 1)) * A.B + (long long)(il - 1) * A.nt + term;
}

// Local force on every local node of every subdomain (src/sg.cpp:252-293):
//   f_k = M (um_k + a0 uc_k) + a1 sum G_ijk K_i uc_j  (+ f_ext on k = 0,
//   weighted by D_s on the interface).  Interior rows -> yI (block-row layout),
//   interface rows -> fG (LI layout).
__global__ void local_force_kernel(LocalArgs A, int n, const double* __restrict__ um, const double* __restrict__ uc,
                                   double a0, double a1, const double* __restrict__ fnext, int fdof, double fval,
                                   const double* __restrict__ iface_w, const int* __restrict__ ip_off,
                                   double* __restrict__ yI, double* __restrict__ fG, int ns,
                                   const int* __restrict__ list, long long nlist) {
  // all local nodes, or only the (s * nl + lid) entries of `list`
  const long long total = list ? nlist * A.nt : (long long)ns * A.nl * A.nt;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int lid, k, s;
    if (list) {
      // term-major: a warp's lanes share the output term k (uniform loops over
      // its tensor entries, broadcast entry loads) and cover consecutive nodes
      const int e = list[t % nlist];
      s = e / A.nl, lid = e % A.nl, k = int(t / nlist);
    } else {
      lid = int(t % A.nl), k = int((t / A.nl) % A.nt), s = int(t / ((long long)A.nl * A.nt));
    }
    const int cls = A.lid_to_p[(long long)s * A.nl + lid];
    if (cls == -1) continue;  // Dirichlet node
    const int il = lid % (A.mx + 1), jl = lid / (A.mx + 1);
    const double* Ms = A.Ml + (long long)s * 4 * A.nl;
    const double* Ks = A.Kl + (long long)s * A.nin * 3 * A.nl;
    int nbl[7], nbd[7];
#pragma unroll
    for (int dir = 0; dir < 7; ++dir) {
      const int i2 = il + sDI[dir], j2 = jl + sDJ[dir];
      const bool in = i2 >= 0 && i2 <= A.mx && j2 >= 0 && j2 <= A.my;
      nbl[dir] = in ? j2 * (A.mx + 1) + i2 : lid;
      nbd[dir] = (in && A.lid_to_p[(long long)s * A.nl + nbl[dir]] != -1) ? lid_dof(A, s, i2, j2) : -1;
    }
    double f = 0.0;
#pragma unroll
    for (int dir = 0; dir < 7; ++dir)
      if (nbd[dir] >= 0) {
        const long long o = (long long)k * n + nbd[dir];
        f += mco(Ms, A.nl, lid, nbl[dir], dir) * (um[o] + a0 * uc[o]);
      }
    if (a1 > 0.0) {
      for (int e = A.g.ptr[k]; e < A.g.ptr[k + 1]; ++e) {
        const double* Ki = Ks + (long long)A.g.i[e] * 3 * A.nl;
        const double* xj = uc + (long long)A.g.j[e] * n;
        double sacc = 0.0;
#pragma unroll
        for (int dir = 0; dir < 5; ++dir)
          if (nbd[dir] >= 0) sacc += kco(Ki, A.nl, lid, nbl[dir], dir) * xj[nbd[dir]];
        f += (a1 * A.g.v[e]) * sacc;
      }
    }
    const int mydof = nbd[0];
    const double wgt = cls >= 0 ? iface_w[ip_off[s] + cls] : 1.0;
    if (k == 0) {
      if (fnext) f += wgt * fnext[mydof];
      else if (mydof == fdof) f += wgt * fval;
    }
    if (cls == -2)
      yI[interior_index(A, s, il, jl, k)] = f;
    else
      fG[A.lioff[s] + (long long)k * A.ng[s] + cls] = f;
  }
}

// Transient-operator product restricted to couplings between node classes.
//  mode 0 (A_GI y):  out_LI[s][k*ng+p] = fG - sum_{interior nb} A(p,nb) y(nb)
//  mode 1 (A_IG u):  out_I[s][..]      = sum_{interface nb} A(lid,nb) uLI(nb)
//  mode 2 (S u):     out_LI[s][k*ng+p] = sum_{interface nb, self} A(p,nb) uLI(nb)
//                                        - sum_{interior nb} A(p,nb) y(nb)
//                    (y = A_II^-1 A_IG u: the implicit local Schur product)
__global__ void coupling_kernel(LocalArgs A, int mode, const double* __restrict__ yI, const double* __restrict__ fG,
                                const double* __restrict__ uLI, const int* __restrict__ ip_off,
                                const int* __restrict__ iface_lid, double* __restrict__ outLI,
                                double* __restrict__ outI, int ns, const int* __restrict__ list, long long nlist) {
  const long long total = list ? nlist * A.nt : (long long)ns * A.nl * A.nt;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int lid, k, s;
    if (list) {
      const int e = list[t / A.nt];
      s = e / A.nl, lid = e % A.nl, k = int(t % A.nt);
    } else {
      lid = int(t % A.nl), k = int((t / A.nl) % A.nt), s = int(t / ((long long)A.nl * A.nt));
    }
    const int cls = A.lid_to_p[(long long)s * A.nl + lid];
    if (mode == 1 ? cls != -2 : cls < 0) continue;
    const int il = lid % (A.mx + 1), jl = lid / (A.mx + 1);
    const double* Ms = A.Ml + (long long)s * 4 * A.nl;
    const double* Ks = A.Kl + (long long)s * A.nin * 3 * A.nl;
    const int ng = A.ng[s];
    double acc = 0.0;
    for (int dir = mode == 2 ? 0 : 1; dir < 7; ++dir) {
      const int i2 = il + sDI[dir], j2 = jl + sDJ[dir];
      if (i2 < 0 || i2 > A.mx || j2 < 0 || j2 > A.my) continue;
      const int nb = j2 * (A.mx + 1) + i2;
      const int c2 = A.lid_to_p[(long long)s * A.nl + nb];
      if (mode == 0 ? c2 != -2 : mode == 1 ? c2 < 0 : c2 == -1) continue;
      // value of the other node for term j (mode 2: interface u, interior -y)
      auto val = [&](int j) -> double {
        if (mode == 0 || (mode == 2 && c2 == -2)) {
          const double y = yI[interior_index(A, s, i2, j2, j)];
          return mode == 0 ? y : -y;
        }
        return uLI[A.lioff[s] + (long long)j * ng + c2];
      };
      acc += A.ms * mco(Ms, A.nl, lid, nb, dir) * val(k);
      if (dir < 5)
        for (int e = A.g.ptr[k]; e < A.g.ptr[k + 1]; ++e)
          acc += (A.ss * A.g.v[e]) * kco(Ks + (long long)A.g.i[e] * 3 * A.nl, A.nl, lid, nb, dir) * val(A.g.j[e]);
    }
    if (mode == 0) {
      const long long o = A.lioff[s] + (long long)k * ng + cls;
      outLI[o] = fG[o] - acc;
    } else if (mode == 2) {
      outLI[A.lioff[s] + (long long)k * ng + cls] = acc;
    } else {
      outI[interior_index(A, s, il, jl, k)] = acc;
    }
  }
}

// ----------------------------------------------------- coupling blocks ---
// Block of the transient operator between interface node q and interior node
// i of subdomain s (direction dir from q):  C[k][j] = ms M(q,i) d_kj +
// ss sum_{(i', j, g) in G(k)} g K_i'(q, i)  -- symmetric, and A(i, q) = A(q, i).
// One CTA per edge, thread = row k.
__global__ void coupling_block_kernel(LocalArgs A, const int4* __restrict__ edge, double* __restrict__ blk) {
  const int4 e = edge[blockIdx.x];
  const int s = e.x, q = e.y, nb = e.z, dir = e.w, nt = A.nt;
  const double* Ms = A.Ml + (long long)s * 4 * A.nl;
  const double* Ks = A.Kl + (long long)s * A.nin * 3 * A.nl;
  double* C = blk + (long long)blockIdx.x * nt * nt;
  const double m = A.ms * mco(Ms, A.nl, q, nb, dir);
  for (int k = threadIdx.x; k < nt; k += blockDim.x) {
    double* row = C + (long long)k * nt;
    for (int j = 0; j < nt; ++j) row[j] = j == k ? m : 0.0;
    if (dir < 5)
      for (int g = A.g.ptr[k]; g < A.g.ptr[k + 1]; ++g)
        row[A.g.j[g]] += (A.ss * A.g.v[g]) * kco(Ks + (long long)A.g.i[g] * 3 * A.nl, A.nl, q, nb, dir);
  }
}

// mode 0 (A_GI y): out_LI[s][k ng + p] = fG - sum_{edges of q} C y(i)
// mode 1 (A_IG u): out_I[s][..]      = sum_{edges of i} C u(q)
// thread = (list entry, k), node-major: the lanes of a node share its edges
__global__ void coupling_blk_kernel(LocalArgs A, int mode, const double* __restrict__ blk,
                                    const int4* __restrict__ edge, const int* __restrict__ q_cls,
                                    const int* __restrict__ ptr, const int* __restrict__ eidx,
                                    const int* __restrict__ list, long long nlist, const double* __restrict__ yI,
                                    const double* __restrict__ fG, const double* __restrict__ uLI,
                                    double* __restrict__ outLI, double* __restrict__ outI) {
  const int nt = A.nt;
  const int total = int(nlist) * nt;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int a = t / nt, k = t % nt;
    double acc = 0.0;
    for (int c = ptr[a]; c < ptr[a + 1]; ++c) {
      const int ed = eidx[c];
      const int4 e = edge[ed];
      const double* row = blk + ((long long)ed * nt + k) * nt;
      if (mode == 0) {
        const int i2 = e.z % (A.mx + 1), j2 = e.z / (A.mx + 1);
        const double* y = yI + ((long long)e.x * A.H + (j2 - 1)) * A.B + (long long)(i2 - 1) * nt;
        for (int j = 0; j < nt; ++j) acc = fma(__ldg(row + j), y[j], acc);
      } else {
        const double* u = uLI + A.lioff[e.x] + q_cls[ed];
        const int ng = A.ng[e.x];
        for (int j = 0; j < nt; ++j) acc = fma(__ldg(row + j), u[(long long)j * ng], acc);
      }
    }
    const int en = list[a], s = en / A.nl, lid = en % A.nl;
    if (mode == 0) {
      const long long o = A.lioff[s] + (long long)k * A.ng[s] + A.lid_to_p[(long long)s * A.nl + lid];
      outLI[o] = fG[o] - acc;
    } else {
      outI[interior_index(A, s, lid % (A.mx + 1), lid / (A.mx + 1), k)] = acc;
    }
  }
}

// Stiffness part of the local force on the interface list, per (entry a,
// direction d <= 4): B[k][j] = sum_{(i, j, g) in G(k)} g K_i(q, nb_d) (the
// element-assembled stencil of q; scaled by alpha1 at use).  CTA per (a, d).
__global__ void force_block_kernel(LocalArgs A, const int* __restrict__ list, double* __restrict__ blk) {
  const int a = blockIdx.x / 5, dir = blockIdx.x % 5, nt = A.nt;
  const int e = list[a], s = e / A.nl, q = e % A.nl;
  const int il = q % (A.mx + 1), jl = q / (A.mx + 1);
  const int i2 = il + sDI[dir], j2 = jl + sDJ[dir];
  const bool in = i2 >= 0 && i2 <= A.mx && j2 >= 0 && j2 <= A.my;
  const int nb = in ? j2 * (A.mx + 1) + i2 : q;
  const double* Ks = A.Kl + (long long)s * A.nin * 3 * A.nl;
  double* C = blk + (long long)blockIdx.x * nt * nt;
  for (int k = threadIdx.x; k < nt; k += blockDim.x) {
    double* row = C + (long long)k * nt;
    for (int j = 0; j < nt; ++j) row[j] = 0.0;
    if (in)
      for (int g = A.g.ptr[k]; g < A.g.ptr[k + 1]; ++g)
        row[A.g.j[g]] += A.g.v[g] * kco(Ks + (long long)A.g.i[g] * 3 * A.nl, A.nl, q, nb, dir);
  }
}

// local_force_kernel's interface rows with the stiffness part from the blocks
__global__ void local_force_blk_kernel(LocalArgs A, int n, const double* __restrict__ um, const double* __restrict__ uc,
                                       double a0, double a1, const double* __restrict__ fnext, int fdof, double fval,
                                       const double* __restrict__ iface_w, const int* __restrict__ ip_off,
                                       double* __restrict__ fG, const int* __restrict__ list, long long nlist,
                                       const double* __restrict__ blk) {
  const int nt = A.nt, total = int(nlist) * nt;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int a = t / nt, k = t % nt;
    const int e = list[a], s = e / A.nl, lid = e % A.nl;
    const int cls = A.lid_to_p[(long long)s * A.nl + lid];
    const int il = lid % (A.mx + 1), jl = lid / (A.mx + 1);
    const double* Ms = A.Ml + (long long)s * 4 * A.nl;
    double f = 0.0;
    int nbd0 = -1;
#pragma unroll
    for (int dir = 0; dir < 7; ++dir) {
      const int i2 = il + sDI[dir], j2 = jl + sDJ[dir];
      if (i2 < 0 || i2 > A.mx || j2 < 0 || j2 > A.my) continue;
      const int nbl = j2 * (A.mx + 1) + i2;
      if (A.lid_to_p[(long long)s * A.nl + nbl] == -1) continue;
      const int nbd = lid_dof(A, s, i2, j2);
      if (dir == 0) nbd0 = nbd;
      const long long o = (long long)k * n + nbd;
      f += mco(Ms, A.nl, lid, nbl, dir) * (um[o] + a0 * uc[o]);
      if (dir < 5 && a1 > 0.0) {
        const double* row = blk + (((long long)a * 5 + dir) * nt + k) * nt;
        double sacc = 0.0;
        for (int j = 0; j < nt; ++j) sacc = fma(__ldg(row + j), uc[(long long)j * n + nbd], sacc);
        f += a1 * sacc;
      }
    }
    const double wgt = iface_w[ip_off[s] + cls];
    if (k == 0) {
      if (fnext) f += wgt * fnext[nbd0];
      else if (nbd0 == fdof) f += wgt * fval;
    }
    fG[A.lioff[s] + (long long)k * A.ng[s] + cls] = f;
  }
}

void GpuSolver::build_coupling_blocks() {
  // edges from the interface list (A_GI rows) and their transposes for the
  // interior list (A_IG rows); host copies of the lists and classes
  std::vector<int> il(n_ilist_), al(n_alist_), cls((size_t)NS * G.nl);
  if (n_ilist_) SGW_CUDA(cudaMemcpy(il.data(), ilist_.p, il.size() * sizeof(int), cudaMemcpyDeviceToHost));
  if (n_alist_) SGW_CUDA(cudaMemcpy(al.data(), alist_.p, al.size() * sizeof(int), cudaMemcpyDeviceToHost));
  SGW_CUDA(cudaMemcpy(cls.data(), lid_to_p.p, cls.size() * sizeof(int), cudaMemcpyDeviceToHost));
  static const int DI[7] = {0, 1, -1, 0, 0, 1, -1}, DJ[7] = {0, 0, 0, 1, -1, 1, -1};
  const int w = G.mx + 1;
  std::vector<int4> edges;
  std::vector<int> qcls, iptr(1, 0), iedge;
  std::vector<std::vector<int>> by_interior((size_t)NS * G.nl);
  for (size_t a = 0; a < il.size(); ++a) {
    const int s = il[a] / G.nl, q = il[a] % G.nl, i0 = q % w, j0 = q / w;
    for (int dir = 1; dir < 7; ++dir) {
      const int i2 = i0 + DI[dir], j2 = j0 + DJ[dir];
      if (i2 < 0 || i2 > G.mx || j2 < 0 || j2 > G.my) continue;
      const int nb = j2 * w + i2;
      if (cls[(size_t)s * G.nl + nb] != -2) continue;
      by_interior[(size_t)s * G.nl + nb].push_back((int)edges.size());
      iedge.push_back((int)edges.size());
      edges.push_back(make_int4(s, q, nb, dir));
      qcls.push_back(cls[(size_t)s * G.nl + q]);
    }
    iptr.push_back((int)iedge.size());
  }
  std::vector<int> aptr(1, 0), aedge;
  for (int e : al) {
    for (int ed : by_interior[e]) aedge.push_back(ed);
    aptr.push_back((int)aedge.size());
  }
  cpl_edge_.upload(edges), cpl_q_cls_.upload(qcls), cpl_iptr_.upload(iptr), cpl_iedge_.upload(iedge);
  cpl_aptr_.upload(aptr), cpl_aedge_.upload(aedge);
  // Built once at setup and only while they leave >= 1 GiB free: without them
  // the step uses the stencil kernels (coupling_kernel / local_force_kernel),
  // which need no extra memory.  Reduced-memory mode skips the force blocks.
  auto fits = [&](size_t bytes) {
    if (std::getenv("SGW_NO_CPL_BLOCKS")) return false;  // test hook: the stencil kernels
    size_t fr = 0, tot = 0;
    SGW_CUDA(cudaMemGetInfo(&fr, &tot));
    return bytes + (size_t(1) << 30) <= fr;
  };
  auto try_alloc = [&](DBuf<double>& b, size_t count) {
    if (!fits(count * sizeof(double))) return false;
    try {
      b.alloc(count);
      return true;
    } catch (const Error&) {
      (void)cudaGetLastError();
      return false;
    }
  };
  const size_t cb = edges.size() * (size_t)NT * NT;
  if (cb > 0 && try_alloc(cpl_blk_, cb)) {
    coupling_block_kernel<<<(unsigned)edges.size(), 32, 0, st_>>>(local_args(), cpl_edge_.p, cpl_blk_.p);
    SGW_LAUNCHED();
  }
  // local-force stiffness blocks of the interface list
  const size_t fb = (size_t)n_ilist_ * 5 * NT * NT;
  if (fb > 0 && !P.implicit_schur && fb * sizeof(double) <= (size_t(4) << 30) && try_alloc(frc_blk_, fb)) {
    force_block_kernel<<<(unsigned)(n_ilist_ * 5), 32, 0, st_>>>(local_args(), ilist_.p, frc_blk_.p);
    SGW_LAUNCHED();
  }
  cpl_built_ = true;
}

// --------------------------------------------------------------- Newmark ---
__global__ void predictor_kernel(const double* __restrict__ u, const double* __restrict__ v,
                                 const double* __restrict__ a, double* __restrict__ um, double* __restrict__ uc,
                                 long long N, double dt, double zeta, double gamma) {
  const double zdd = zeta * dt * dt, c1 = (1.0 - 2.0 * zeta) / (2.0 * zeta);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const double m = (u[i] + dt * v[i]) / zdd + c1 * a[i];  // src/newmark.cpp:16-20
    um[i] = m;
    uc[i] = gamma * dt * m - v[i] - (1.0 - gamma) * dt * a[i];  // :22-26
  }
}

// u_next from the interface solution and the recovered interiors, then the
// Newmark update (src/sg.cpp:334-354, src/newmark.cpp:39-49).
__global__ void update_kernel(double* __restrict__ u, double* __restrict__ v, double* __restrict__ a,
                              const double* __restrict__ ug, const double* __restrict__ yI,
                              const double* __restrict__ wI, const int* __restrict__ iface_of_dof, int n, int nt,
                              int n_iface, int nx, int ny, int px, int py, int H, int B,
                              const int* __restrict__ gid_local, double dt, double zeta, double gamma,
                              const int* __restrict__ conv) {
  // conv: the persistent PCG's convergence flag; an unconverged solve leaves the
  // state untouched (the reference throws before newmark_update, sg.cpp:412-416)
  if (conv && *conv == 0) return;
  const int N = n * nt;  // < 2^31 (GpuSolver ctor): 32-bit derived indices
  const double zdd = zeta * dt * dt, c1 = (1.0 - 2.0 * zeta) / (2.0 * zeta);
  // 64-bit loop variable: t + stride must not overflow near N = 2^31 - 1
  for (long long tt = blockIdx.x * (long long)blockDim.x + threadIdx.x; tt < N; tt += (long long)gridDim.x * blockDim.x) {
    const int t = int(tt), d = t % n, k = t / n;
    const int q = iface_of_dof[d];
    double un;
    if (q >= 0) {
      un = ug[(long long)k * n_iface + q];
    } else {
      const int gi = d % (nx - 1) + 1, gj = d / (nx - 1) + 1;
      // interior node: cell gi lies in the same block (partition.cpp:70-76)
      const int sx = gi * px / nx, sy = gj * py / ny;
      const int il = gi - block_origin(sx, nx, px), jl = gj - block_origin(sy, ny, py);
      const int sl = gid_local[sy * px + sx];
      if (sl < 0) continue;  // sharded: interior of another rank's subdomain
      const long long idx = ((long long)sl * H + (jl - 1)) * B + (long long)(il - 1) * nt + k;
      un = yI[idx] - wI[idx];
    }
    const double uo = u[t], vo = v[t], ao = a[t];
    const double an = (un - uo - dt * vo) / zdd - c1 * ao;
    v[t] = vo + (1.0 - gamma) * dt * ao + gamma * dt * an;
    a[t] = an;
    u[t] = un;
  }
}

__global__ void probe_kernel(const double* __restrict__ u, const int* __restrict__ pd, const int* __restrict__ own,
                             int np, int n, int nt, double* __restrict__ out, const int* __restrict__ conv) {
  if (conv && *conv == 0) return;  // unconverged step: no new history row
  // per probe: mean, std, then every chaos coefficient u_0 .. u_P (sg.cpp:391-405)
  for (int p = threadIdx.x; p < np; p += blockDim.x) {
    double* o = out + (long long)p * (2 + nt);
    if (own && !own[p]) {  // sharded: the owning rank contributes this probe
      for (int j = 0; j < 2 + nt; ++j) o[j] = 0.0;
      continue;
    }
    double var = 0.0;
    for (int j = 1; j < nt; ++j) {
      const double c = u[(long long)j * n + pd[p]];
      var += c * c;
    }
    o[0] = u[pd[p]];
    o[1] = sqrt(var);
    for (int j = 0; j < nt; ++j) o[2 + j] = u[(long long)j * n + pd[p]];
  }
}

__global__ void reduce_nodal_kernel(const double* __restrict__ nodal, double* __restrict__ out, int nx, int ny) {
  const int n = (nx - 1) * (ny - 1);
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    const int gi = d % (nx - 1) + 1, gj = d / (nx - 1) + 1;
    out[d] = nodal[gj * (nx + 1) + gi];
  }
}

__global__ void axpby_kernel(double* __restrict__ y, const double* __restrict__ x, long long N, double a, double b) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
    y[i] = a * y[i] + b * x[i];
}
__global__ void cg_mass_update(double* __restrict__ x, double* __restrict__ r, double* __restrict__ p,
                               const double* __restrict__ q, const double* __restrict__ z, long long N, double alpha) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    r[i] -= alpha * q[i];
  }
}

// res = ((f0 - a0 M v) - a1 K v) - K u   (src/sg.cpp:367-369)
__global__ void init_resid_kernel(double* __restrict__ res, const double* __restrict__ mv,
                                  const double* __restrict__ kv, const double* __restrict__ ku, long long N,
                                  double a0, double a1) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
    res[i] = res[i] - a0 * mv[i] - a1 * kv[i] - ku[i];
}

// Reduced-memory Schur product: y = sum_s R_s^T (A_GG,s -
// A_GI,s A_II,s^-1 A_IG,s) R_s x with the subdomains' local stencils and one
// batched interior sweep, instead of the stored dense S_s (dd.cpp:142-157 on
// the S of sg.cpp:227-245).  Scratch: li_x (x local), wI (interior), li_y.
void GpuSolver::schur_matvec_implicit(const double* x, double* y) {
  const LocalArgs A = local_args();
  const long long ti = (long long)n_ilist_ * NT, ta = (long long)n_alist_ * NT;
  gather_li(x, li_x.p, false);
  SGW_CUDA(cudaMemsetAsync(wI.p, 0, wI.n * sizeof(double), st_));
  if (n_alist_ > 0) {
    coupling_kernel<<<std::max(1, std::min(cdiv(ta, 128), 65535)), 128, 0, st_>>>(
        A, 1, nullptr, nullptr, li_x.p, ip_off.p, iface_lid_.p, nullptr, wI.p, NS, alist_.p, n_alist_);
    SGW_LAUNCHED();
  }
  sweep(wI.p);  // A_II^-1 A_IG x
  coupling_kernel<<<std::max(1, std::min(cdiv(ti, 128), 65535)), 128, 0, st_>>>(
      A, 2, wI.p, nullptr, li_x.p, ip_off.p, iface_lid_.p, li_y.p, nullptr, NS, ilist_.p, n_ilist_);
  SGW_LAUNCHED();
  scatter_li(li_y.p, y, false, nullptr, nullptr);
  halo_sum(y);
}

// ---------------------------------------------------------------- driver ---
void GpuSolver::set_force_point(int node, double f0, double t0, double amp) {
  force_kind_ = node >= 0 ? 1 : 0;
  force_node_ = node;
  const int gi = node % (P.nx + 1), gj = node / (P.nx + 1);
  force_dof_ = node >= 0 ? G.dof(gi, gj) : -1;
  force_f0_ = f0, force_t0_ = t0, force_amp_ = amp;
}

void GpuSolver::set_force_table(const double* table, int rows) {
  force_kind_ = 2;
  // sgw_run is synchronous: the caller's table outlives every step, so rows are
  // uploaded straight from it (no host copy of the table)
  force_tab_ = table;
  force_len_ = (size_t)rows * P.n_nodes();
  if (force_row_.n != (size_t)P.n_nodes()) force_row_.alloc(P.n_nodes());
  if (fext_.n != (size_t)n) fext_.alloc(n);
}

static double ricker(double t, double f0, double t0, double amp) {
  const double a = M_PI * M_PI * f0 * f0 * (t - t0) * (t - t0);
  return amp * (1.0 - 2.0 * a) * std::exp(-a);
}

// Force at time t as a reduced vector (kind 2) or a point value (kind 1).
const double* GpuSolver::force_at(double t, int row, double* fval) {
  *fval = 0.0;
  if (force_kind_ == 1) {
    *fval = force_dof_ >= 0 ? ricker(t, force_f0_, force_t0_, force_amp_) : 0.0;
    return nullptr;
  }
  if (force_kind_ == 2) {
    const size_t nn = P.n_nodes();
    if ((size_t)row * nn >= force_len_) throw Error(1, "force table too short");
    SGW_CUDA(cudaMemcpyAsync(force_row_.p, force_tab_ + (size_t)row * nn, nn * sizeof(double),
                             cudaMemcpyHostToDevice, st_));
    reduce_nodal_kernel<<<cdiv(n, 256), 256, 0, st_>>>(force_row_.p, fext_.p, P.nx, P.ny);
    SGW_LAUNCHED();
    return fext_.p;
  }
  return nullptr;
}

LocalArgs GpuSolver::local_args() const {
  return LocalArgs{Kl.p, Ml.p, GList{gk_ptr.p, gk_i.p, gk_j.p, gk_v.p}, lid_to_p.p, Sp.d_xoff.p, ng_d.p, sub_gid_d_.p,
                   G.nl, NIN, NT, G.mx, G.my, G.px, P.nx, G.py, P.ny, G.H, B, P.mass_scale, P.stiff_scale};
}

// src/sg.cpp:358-376: u, v in block 0, a = M^-1 (f0 - a0 M v - a1 K v - K u).
void GpuSolver::init_state(const double* u0_nodal, const double* v0_nodal, double) {
  u.zero(st_), v.zero(st_), a.zero(st_);
  reduce_nodal_kernel<<<cdiv(n, 256), 256, 0, st_>>>(u0_nodal, u.p, P.nx, P.ny);
  SGW_LAUNCHED();
  reduce_nodal_kernel<<<cdiv(n, 256), 256, 0, st_>>>(v0_nodal, v.p, P.nx, P.ny);
  SGW_LAUNCHED();
  t_now = 0.0;
  step_index = 0;
  rhs_ahead_ = false;
  // resid = f0 - a0 M v - a1 K v - K u
  // work vectors kept across runs (a cudaMalloc / cudaFree per run would synchronise)
  if (init_w_.n != 4 * NSTATE) init_w_.alloc(4 * NSTATE);
  struct { double* p; } mv{init_w_.p}, kv{init_w_.p + NSTATE}, ku{init_w_.p + 2 * NSTATE}, res{init_w_.p + 3 * NSTATE};
  apply_block(0, v.p, mv.p);
  apply_block(1, v.p, kv.p);
  apply_block(1, u.p, ku.p);
  SGW_CUDA(cudaMemsetAsync(res.p, 0, NSTATE * sizeof(double), st_));
  double fval = 0.0;
  const double* fvec = force_at(0.0, 0, &fval);
  if (fvec)
    SGW_CUDA(cudaMemcpyAsync(res.p, fvec, n * sizeof(double), cudaMemcpyDeviceToDevice, st_));
  else if (force_kind_ == 1 && force_dof_ >= 0)
    SGW_CUDA(cudaMemcpyAsync(res.p + force_dof_, &fval, sizeof(double), cudaMemcpyHostToDevice, st_));
  init_resid_kernel<<<cdiv((long long)NSTATE, 256), 256, 0, st_>>>(res.p, mv.p, kv.p, ku.p, (long long)NSTATE,
                                                                    P.alpha0, P.alpha1);
  SGW_LAUNCHED();
  mass_solve(a.p, res.p);
  SGW_CUDA(cudaStreamSynchronize(st_));
}

void GpuSolver::record_probes(int k, const int* conv) {
  if (probe_dofs.empty() || k >= probe_cap) return;
  const size_t w = probe_dofs.size() * (2 + NT);
  double* row = probe_hist.p + (size_t)k * w;
  probe_kernel<<<1, 128, 0, st_>>>(u.p, d_probe_dofs.p, comm_ ? d_probe_own.p : nullptr, (int)probe_dofs.size(), n,
                                   NT, row, conv);
  SGW_LAUNCHED();
  allreduce(row, w);
}

__global__ void mask_state_kernel(double* __restrict__ x, const double* __restrict__ mask, int n, long long N) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
    x[i] *= mask[i % n];
}

void GpuSolver::gather_state(double* dst) {
  SGW_CUDA(cudaMemcpyAsync(dst, u.p, NSTATE * sizeof(double), cudaMemcpyDeviceToDevice, st_));
  if (!comm_) return;
  if (own_mask_.n != (size_t)n) {
    std::vector<double> m(n);
    for (int d = 0; d < n; ++d) m[d] = G.owner_of_dof(d) == comm_->rank() ? 1.0 : 0.0;
    own_mask_.upload(m);
  }
  mask_state_kernel<<<std::min(cdiv((long long)NSTATE, 256), 4096), 256, 0, st_>>>(dst, own_mask_.p, n,
                                                                                   (long long)NSTATE);
  SGW_LAUNCHED();
  allreduce(dst, NSTATE);
}

// Interior rows of the local force from the global operator: the stencil of a
// subdomain-interior node only touches that subdomain's elements, so its local
// row equals the global row (f_ext added on term 0, weight 1).
// The JIT operator's y = a0 M uc + a1 sum c K uc arrives in yg; the mass term
// of um (M um_k, a 7-point stencil) is added here, where the loads are cheap.
__global__ void interior_from_global_kernel(LocalArgs A, int n, const double* __restrict__ yg,
                                            const double* __restrict__ Mg, const double* __restrict__ um,
                                            const double* __restrict__ fnext, int fdof, double fval,
                                            double* __restrict__ yI, int ns) {
  const int total = ns * A.H * A.B;  // < 2^31 (GpuSolver ctor)
  const int rw = A.nx - 1, rh = A.ny - 1;
  for (long long tt = blockIdx.x * (long long)blockDim.x + threadIdx.x; tt < total;
       tt += (long long)gridDim.x * blockDim.x) {
    const int t = int(tt);
    const int row = t % A.B, jl = (t / A.B) % A.H + 1, s = t / (A.B * A.H);
    const int il = row / A.nt + 1, k = row % A.nt;
    const int lid = jl * (A.mx + 1) + il;
    if (A.lid_to_p[(long long)s * A.nl + lid] != -2) continue;  // unit row of a ragged block
    const int d = lid_dof(A, s, il, jl);
    const int gi = d % rw, gj = d / rw;
    const double* uk = um + (long long)k * n;
    double q = 0.0;
#pragma unroll
    for (int dir = 0; dir < 7; ++dir) {
      const int i2 = gi + sDI[dir], j2 = gj + sDJ[dir];
      if (i2 >= 0 && i2 < rw && j2 >= 0 && j2 < rh) {
        const int nb = j2 * rw + i2;
        q += mco(Mg, n, d, nb, dir) * __ldg(uk + nb);
      }
    }
    double f = yg[(long long)k * n + d] + q;
    if (k == 0) {
      if (fnext) f += fnext[d];
      else if (d == fdof) f += fval;
    }
    yI[t] = f;
  }
}

// Right-hand-side phase of the step that ends at time t_next (force row
// row_next): predictors, local force, interior solve y = A_II^-1 f_I and the
// interface right-hand side g.  It reads the state (u, v, a) and writes scratch
// only, so step() may put it on the stream for the following step before it has
// read the current step's verdict.
void GpuSolver::launch_rhs(double t_next, int row_next, cudaEvent_t e0, cudaEvent_t e1) {
  const long long N = (long long)NSTATE;
  const int grid = std::min(cdiv(N, 256), 8 * kNumSMs * 8);
  nvtxRangePushA("rhs: predictors, local force, interior solve, interface assembly");
  cudaEventRecord(e0, st_);
  predictor_kernel<<<grid, 256, 0, st_>>>(u.p, v.p, a.p, um.p, uc.p, N, P.dt, P.zeta, P.gamma);
  SGW_LAUNCHED();
  double fval = 0.0;
  const double* fvec = force_at(t_next, row_next, &fval);
  const LocalArgs A = local_args();
  const long long tl = (long long)NS * G.nl * NT;
  const int fdof = force_kind_ == 1 ? force_dof_ : -1;
  const long long ti = (long long)n_ilist_ * NT;
  if (sgop_) {
    // interior rows: f = M um + a0 M uc + a1 sum c K uc on the global grid (JIT
    // operator), copied into the block rows; interface rows: local stencils
    SgOpArgs sa = sgop_args_;
    sa.x = uc.p, sa.y = yglob_.p;  // + M um in interior_from_global_kernel
    sa.alpha = P.alpha0, sa.beta = P.alpha1;
    {
      cudaEvent_t e;
      KP.begin(K_SGOP, st_, &e);
      launch_sgop(*sgop_, sa, st_);
      KP.end(st_);
    }
    const long long tI = (long long)NS * G.H * B;
    interior_from_global_kernel<<<std::min(cdiv(tI, 256), 65535), 256, 0, st_>>>(A, n, yglob_.p, Mg.p, um.p, fvec,
                                                                                   fdof, fval, yI.p, NS);
    SGW_LAUNCHED();
    if (frc_blk_.p)
      local_force_blk_kernel<<<std::max(1, std::min(cdiv(ti, 128), 65535)), 128, 0, st_>>>(
          A, n, um.p, uc.p, P.alpha0, P.alpha1, fvec, fdof, fval, iface_w.p, ip_off.p, fG.p, ilist_.p, n_ilist_,
          frc_blk_.p);
    else
      local_force_kernel<<<std::max(1, std::min(cdiv(ti, 128), 65535)), 128, 0, st_>>>(
          A, n, um.p, uc.p, P.alpha0, P.alpha1, fvec, fdof, fval, iface_w.p, ip_off.p, yI.p, fG.p, NS, ilist_.p,
          n_ilist_);
  } else {
    local_force_kernel<<<std::min(cdiv(tl, 256), 65535), 256, 0, st_>>>(
        A, n, um.p, uc.p, P.alpha0, P.alpha1, fvec, fdof, fval, iface_w.p, ip_off.p, yI.p, fG.p, NS, nullptr, 0);
  }
  SGW_LAUNCHED();
  sweep(yI.p);  // y = A_II^-1 f_I
  if (!direct_) {
    if (cpl_blk_.p)
      coupling_blk_kernel<<<std::max(1, std::min(cdiv(ti, 128), 65535)), 128, 0, st_>>>(
          A, 0, cpl_blk_.p, cpl_edge_.p, cpl_q_cls_.p, cpl_iptr_.p, cpl_iedge_.p, ilist_.p, n_ilist_, yI.p, fG.p,
          nullptr, li_y.p, nullptr);
    else  // no room for the coupling blocks: the stencil form
      coupling_kernel<<<std::max(1, std::min(cdiv(ti, 128), 65535)), 128, 0, st_>>>(
          A, 0, yI.p, fG.p, nullptr, ip_off.p, iface_lid_.p, li_y.p, nullptr, NS, ilist_.p, n_ilist_);
    SGW_LAUNCHED();
    scatter_li(li_y.p, vb.p, false, nullptr, nullptr);  // g = sum_s R_s^T g_s
    halo_sum(vb.p);
  }
  nvtxRangePop();
  cudaEventRecord(e1, st_);
}

int GpuSolver::step(int* iters_out, bool more) {
  const long long N = (long long)NSTATE;
  const int grid = std::min(cdiv(N, 256), 8 * kNumSMs * 8);
  NvtxRange nvtx_step("sgw step");
  const LocalArgs A = local_args();
  const long long ta = (long long)n_alist_ * NT;
  // the right-hand-side phase: already on the stream when the previous step launched it ahead
  const cudaEvent_t ev_rhs0 = rhs_par_ ? ev_[8] : ev_[2], ev_rhs1 = rhs_par_ ? ev_[9] : ev_[3];
  if (!rhs_ahead_) launch_rhs(t_now + P.dt, step_index + 1, ev_rhs0, ev_rhs1);
  rhs_ahead_ = false;
  if (direct_) {
    // one subdomain (sg.cpp:301-305): y is the whole solution, no interface solve
    SGW_CUDA(cudaMemsetAsync(wI.p, 0, wI.n * sizeof(double), st_));
    cudaEventRecord(ev_[4], st_);
    update_kernel<<<grid, 256, 0, st_>>>(u.p, v.p, a.p, vx.p, yI.p, wI.p, iface_of_dof.p, n, NT, G.n_iface, P.nx,
                                         P.ny, G.px, G.py, G.H, B, gid_local_d_.p, P.dt, P.zeta, P.gamma, nullptr);
    SGW_LAUNCHED();
    record_probes(step_index + 1, nullptr);
    cudaEventRecord(ev_[5], st_);
    SGW_CUDA(cudaEventSynchronize(ev_[5]));
    t_now = t_now + P.dt;
    ++step_index;
    KP.collect();
    float ms_rhs = 0, ms_all = 0;
    cudaEventElapsedTime(&ms_rhs, ev_rhs0, ev_rhs1);
    cudaEventElapsedTime(&ms_all, ev_rhs0, ev_[5]);
    T.rhs_ms += ms_rhs, T.step_ms += ms_all;
    ++T.steps;
    if (iters_out) *iters_out = 0;
    return 0;
  }
  bool conv = false;
  // persistent PCG: its convergence is read after the recovery is launched
  // (no host round trip between the solve and the rest of the step)
  const bool deferred = fused_ok();
  int it = 0;
  {
    NvtxRange nvtx_pcg("interface PCG (NN2)");
    if (deferred) {
      pcg_fused_launch(vb.p, vx.p);
    } else {
      it = pcg(vb.p, vx.p, &conv, nullptr);
      if (!conv)
        throw Error(3, "stochastic interface solve did not converge at step " + std::to_string(step_index));
    }
  }
  NvtxRange nvtx_rec("recovery: interior solve, Newmark update, probes");
  cudaEventRecord(ev_[4], st_);
  gather_li(vx.p, li_x.p, false);
  // A_IG u_G is non-zero only on interior nodes next to the interface
  SGW_CUDA(cudaMemsetAsync(wI.p, 0, wI.n * sizeof(double), st_));
  if (n_alist_ > 0) {
    if (cpl_blk_.p)
      coupling_blk_kernel<<<std::max(1, std::min(cdiv(ta, 128), 65535)), 128, 0, st_>>>(
          A, 1, cpl_blk_.p, cpl_edge_.p, cpl_q_cls_.p, cpl_aptr_.p, cpl_aedge_.p, alist_.p, n_alist_, nullptr,
          nullptr, li_x.p, nullptr, wI.p);
    else
      coupling_kernel<<<std::max(1, std::min(cdiv(ta, 128), 65535)), 128, 0, st_>>>(
          A, 1, nullptr, nullptr, li_x.p, ip_off.p, iface_lid_.p, nullptr, wI.p, NS, alist_.p, n_alist_);
    SGW_LAUNCHED();
  }
  sweep(wI.p);  // A_II^-1 A_IG u_G
  update_kernel<<<grid, 256, 0, st_>>>(u.p, v.p, a.p, vx.p, yI.p, wI.p, iface_of_dof.p, n, NT, G.n_iface, P.nx,
                                       P.ny, G.px, G.py, G.H, B, gid_local_d_.p, P.dt, P.zeta, P.gamma,
                                       deferred ? fused_out_.p + 1 : nullptr);
  SGW_LAUNCHED();
  record_probes(step_index + 1, deferred ? fused_out_.p + 1 : nullptr);
  cudaEventRecord(ev_[5], st_);
  const size_t kp_own = KP.mark();
  static const bool no_ahead = std::getenv("SGW_NO_RHS_AHEAD") != nullptr;  // comparison hook
  if (more && deferred && !no_ahead) {
    // keep the GPU busy while the host reads this step's verdict: the next
    // step's right-hand side only reads the state and writes scratch, so after
    // a non-converged solve (state un-advanced on device) it is simply dropped
    launch_rhs((t_now + P.dt) + P.dt, step_index + 2, rhs_par_ ? ev_[2] : ev_[8], rhs_par_ ? ev_[3] : ev_[9]);
    rhs_ahead_ = true;
  }
  SGW_CUDA(cudaEventSynchronize(ev_[5]));
  if (deferred) {
    SGW_CUDA(cudaEventSynchronize(ev_[6]));  // the solve's outputs (side stream)
    // the update and the probe row were conditional on the device-side flag:
    // on non-convergence the state, time and step index stay where they were
    it = pcg_fused_finish(&conv, nullptr);
    if (!conv) {
      if (rhs_ahead_) {
        rhs_ahead_ = false;
        SGW_CUDA(cudaStreamSynchronize(st_));
        KP.collect();
      }
      throw Error(3, "stochastic interface solve did not converge at step " + std::to_string(step_index));
    }
  }
  t_now = t_now + P.dt;
  ++step_index;
  KP.collect(kp_own);
  float ms_rhs = 0, ms_rec = 0, ms_all = 0;
  cudaEventElapsedTime(&ms_rhs, ev_rhs0, ev_rhs1);
  cudaEventElapsedTime(&ms_rec, ev_[4], ev_[5]);
  cudaEventElapsedTime(&ms_all, ev_rhs0, ev_[5]);
  if (rhs_ahead_) rhs_par_ ^= 1;
  T.rhs_ms += ms_rhs;
  T.rec_ms += ms_rec;
  T.step_ms += ms_all;
  ++T.steps;
  if (iters_out) *iters_out = it;
  return it;
}

}  // namespace sgw
