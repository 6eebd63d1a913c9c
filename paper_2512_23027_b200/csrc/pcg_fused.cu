// The whole interface PCG solve (src/pcg.cpp:7-50) with the NN2 preconditioner
// (src/dd.cpp:199-253) as ONE persistent cooperative kernel: every CTA walks
// the same phase sequence separated by grid barriers, so a PCG iteration costs
// seven grid barriers instead of a dozen launches plus a host round trip for
// the convergence test.
//
// Per iteration (phase -> grid barrier):
//   1. S tiles      q_tiles(S_s) on p_new = z + beta p gathered on the fly
//   2. S scatter    q = sum_s R_s^T S_s R_s p_new, partial p.q
//   3. update       p = p_new, x += alpha p, r -= alpha q, partial r.r, and the
//                   weighted local copies D_s R_s r (NN2 inputs f_r, f_c)
//   4. Q tiles      Q_s f_r tiles + d_s = f_c - Psi_s^T f_r
//   5. coarse       d = sum_s B_s^T d_s
//   6. coarse solve u_c = F_cc^-1 d
//   7. z scatter    z = sum_s R_s^T D_s [Q f_r - Psi u_c ; u_c], partial r.z
// Reductions: fixed-order block sums, then every CTA sums the block partials
// in index order itself (bitwise identical in every CTA, run to run).
// The convergence test, the true-residual confirmation and the restart from
// the true residual are evaluated on device exactly as src/pcg.cpp:30-40.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "solver.cuh"
#include "tiles.cuh"

namespace cg = cooperative_groups;

namespace sgw {

// A TilePack walked in contiguous tile ranges, one per CTA (tiles are ordered
// matrix by matrix, row-major over the lower tiles (I, J <= I)).  A CTA keeps
// the local input vector of its current matrix and a local accumulator in
// shared memory, adds every tile's row and column products into it, and at
// a matrix boundary writes the accumulator as its partial of that matrix:
// y_s = sum over the CTAs covering s of their partials, in CTA order.
struct RangePack {
  const double* tiles;
  const int* nt;              // tiles per side, per matrix
  const long long* xoff;      // local vector offset per matrix (padded, 64 nt)
  const long long* t_first;   // [G + 1] first tile of each CTA's range
  const int4* start;          // [G] {matrix, I, J} of each CTA's first tile
  const int* c0;              // per matrix: first CTA covering it
  const int* ncta;            // per matrix: CTAs covering it
  const long long* pbase;     // per matrix: offset of its partials in part
  double* part;               // partials [pbase[s] + (c - c0[s]) 64 nt[s] + i]
};

struct FusedPcg {
  long long NG, ncol_total;
  int n_iface, NT, NS, n_corner, NC, max_iter, hist_cap;
  double tol;
  const double* b;
  double *x, *r, *z, *p, *q;
  const int4* s_desc;
  const double* s_tiles;
  long long s_ntiles;
  double *s_row, *s_col;
  const long long *s_base, *s_xoff;
  const int *s_nt, *smap;
  const int4* q_desc;
  const double* q_tiles;
  long long q_ntiles;
  double *q_row, *q_col;
  const long long *q_base, *q_xoff;
  const int* q_nt;
  double *fr, *fc;
  const int *inv_cnt, *inv_s, *inv_p, *ip_off, *ng, *nr, *nc, *pkind, *cpos_flat, *cp_off;
  const double* iface_w;
  const int *cinv_cnt, *cinv_s, *cinv_c;
  const long long *roff, *coff, *psioff;
  const double *Psi, *Finv;
  double *dsub, *dco, *uco;
  double* part;  // 8 slots x gridDim
  int* out;      // [0] iterations, [1] converged
  double* hist;  // residual history, hist_cap entries
  const int2 *s_tx, *q_tx;       // per-tile local offsets of the I / J segments
  double *li_z, *li_p, *li_x;    // z, p, x in S-local layout (written by their producers)
  double* tphase;                // 8 accumulated phase times (ns), CTA 0
  double *ucl, *wr;              // B_s u_c (c-space) and Psi_s B_s u_c (r-space, padded)
  long long rlen;                // padded r-space length
  RangePack rs, rq;              // contiguous tile ranges per CTA of S and Q
  int nst, maxlen;               // ring stages; longest local vector (doubles)
  int l2pf;                      // tiles hinted into L2 beyond the ring at a phase switch
  int psi_late;                  // Psi^T f_r after the Q tiles instead of before
};

extern __shared__ __align__(128) double dyn_smem[];  // ring stages, local vector, accumulator

struct Smem {
  double csum[8][kTile];
  double xI[kTile], xJ[kTile];
  double red[40];
};

// Phase clock of CTA 0 / thread 0 (globaltimer, ns): time since the previous
// tick is charged to the phase that just ended (barrier wait included, i.e.
// the critical path).  0 S tiles, 1 S scatter, 2 update, 3 Q tiles + Psi^T,
// 4 coarse assemble, 5 coarse solve, 6 z scatter, 7 init / true residual.
struct PhaseClock {
  bool on;
  unsigned long long last;
  double acc[8];
  __device__ void tick(int ph) {
    if (!on) return;
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    acc[ph] += double(now - last);
    last = now;
  }
};

constexpr int kUnroll = 8;  // independent loads in flight per thread in the glue loops
constexpr int kMaxRing = 8;                    // tile stages per CTA (runtime depth A.nst)
constexpr unsigned kTileBytes = kTile * kTile * 8;

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(su32(b)), "r"(parity)
      : "memory");
}
// Streamed tiles are read once per phase and are far larger than L2: load
// them evict-first so that Psi, F_cc^-1, the partials and the vectors stay
// resident in L2 across phases.
__device__ __forceinline__ void mb_load(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
  asm volatile(
      "{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      " cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(b))
      : "memory");
}

// Per-CTA ring of 32 KB tile stages filled by TMA bulk copies.  The tiles of
// a phase are this CTA's contiguous range; thread 0 keeps nst of them in
// flight.  The matrices are constant, so the next phase's tiles may be issued
// ahead (across grid barriers) whenever the phase is known.
struct Ring {
  double* stage;
  unsigned long long* full;
  int nst;
  int consumed, issued;  // consumed: uniform; issued: thread 0
  int pre_kind;          // tile set whose first tiles are already issued for the next phase
};

__device__ __forceinline__ void ring_issue(Ring& R, const RangePack& P, long long k) {
  const long long t = P.t_first[blockIdx.x] + k;
  if (t >= P.t_first[blockIdx.x + 1]) return;
  const int st = R.issued % R.nst;
  mb_load(R.stage + (size_t)st * kTile * kTile, P.tiles + t * (kTile * kTile), kTileBytes, &R.full[st]);
  ++R.issued;
}
// issue the first tiles of set `kind` for the next tile phase (thread 0),
// and hint the following l2pf tiles into L2 (they stream during glue phases)
__device__ __forceinline__ void ring_prefetch(Ring& R, int kind, const RangePack& P, int l2pf) {
  if (threadIdx.x == 0) {
    for (int n = 0; n < R.nst; ++n) ring_issue(R, P, n);
    const long long t1 = P.t_first[blockIdx.x + 1];
    for (long long t = P.t_first[blockIdx.x] + R.nst, e = t + l2pf; t < e && t < t1; ++t)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.tiles + t * (kTile * kTile)), "r"(kTileBytes)
                   : "memory");
  }
  R.pre_kind = kind;
}

__device__ __forceinline__ double block_total(double v, Smem& sm) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sm.red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = lane < (int)(blockDim.x >> 5) ? sm.red[lane] : 0.0;
    s = warp_sum(s);
  }
  __syncthreads();
  return s;  // valid in thread 0
}

// Deterministic grid sum: block partials, one grid barrier, then every CTA
// adds the partials in index order.
__device__ __forceinline__ double grid_sum(double v, double* part, int slot, cg::grid_group& g, Smem& sm) {
  v = block_total(v, sm);
  if (threadIdx.x == 0) part[(size_t)slot * gridDim.x + blockIdx.x] = v;
  g.sync();
  // all threads load the block totals (<= 2 each), then a fixed-shape block
  // reduction: the same value, bitwise, in every CTA
  double s = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) s += __ldcg(part + (size_t)slot * gridDim.x + b);
  s = block_total(s, sm);
  if (threadIdx.x == 0) sm.red[32] = s;
  __syncthreads();
  const double t = sm.red[32];
  __syncthreads();
  return t;
}

// D_s R_s val for interface flat index q into the NN2 local inputs.
__device__ __forceinline__ void write_local(const FusedPcg& A, long long q, double val) {
  const int j = int(q / A.n_iface), gq = int(q % A.n_iface);
  for (int e = 0; e < A.inv_cnt[gq]; ++e) {
    const int s = A.inv_s[4 * gq + e], pp = A.inv_p[4 * gq + e];
    const int kind = A.pkind[A.ip_off[s] + pp];
    const double wv = A.iface_w[A.ip_off[s] + pp] * val;
    if (kind >= 0) A.fr[A.roff[s] + (long long)j * A.nr[s] + kind] = wv;
    else A.fc[A.coff[s] + (long long)j * A.nc[s] + (-1 - kind)] = wv;
  }
}

// R_s val into an S-local buffer for every subdomain sharing interface index q.
__device__ __forceinline__ void write_local_s(const FusedPcg& A, double* li, long long q, double val) {
  const int j = int(q / A.n_iface), gq = int(q % A.n_iface);
  for (int e = 0; e < A.inv_cnt[gq]; ++e) {
    const int s = A.inv_s[4 * gq + e];
    li[A.s_xoff[s] + (long long)j * A.ng[s] + A.inv_p[4 * gq + e]] = val;
  }
}

// One 64x64 lower tile T_IJ (stage, row-major, diagonal tiles full) times the
// local vector xs: accI += T xs_J, accJ += T^T xs_I (I != J).  256 threads:
// warp w streams rows 8w..8w+7 (128-bit shared loads, lane = 2 columns); the 8
// row sums use a butterfly multi-row reduction, the column sums a shared
// 8 x 64 scratch.  Every accumulator entry has one writer.
__device__ __forceinline__ void tile_acc(const double* T, const double* xI, const double* xJ, bool diag, double* accI,
                                         double* accJ, Smem& sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double2* T2 = reinterpret_cast<const double2*>(T);
  double2 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = T2[(w * 8 + k) * (kTile / 2) + lane];
  const double2 xj = reinterpret_cast<const double2*>(xJ)[lane];
  double rs[8], c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    rs[k] = v[k].x * xj.x + v[k].y * xj.y;
    const double xv = xI[w * 8 + k];
    c0 += v[k].x * xv;
    c1 += v[k].y * xv;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool up = lane & 16;
    const double send = up ? rs[i] : rs[i + 4], keep = up ? rs[i + 4] : rs[i];
    rs[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool up = lane & 8;
    const double send = up ? rs[i] : rs[i + 2], keep = up ? rs[i + 2] : rs[i];
    rs[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const bool up = lane & 4;
    const double send = up ? rs[0] : rs[1], keep = up ? rs[1] : rs[0];
    rs[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  rs[0] += __shfl_xor_sync(0xffffffffu, rs[0], 2);
  rs[0] += __shfl_xor_sync(0xffffffffu, rs[0], 1);
  if ((lane & 3) == 0) {
    const int row = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    accI[w * 8 + row] += rs[0];
  }
  if (!diag) {
    sm.csum[w][2 * lane] = c0;
    sm.csum[w][2 * lane + 1] = c1;
    __syncthreads();
    if (threadIdx.x < kTile) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) s += sm.csum[k][threadIdx.x];
      accJ[threadIdx.x] += s;
    }
  }
}

// write the accumulator as this CTA's partial of matrix s
__device__ __forceinline__ void range_flush(const RangePack& P, int s, int len, const double* acc) {
  double* dst = P.part + P.pbase[s] + (long long)(blockIdx.x - P.c0[s]) * len;
  for (int i = threadIdx.x; i < len; i += blockDim.x) dst[i] = acc[i];
}

// One tile phase over this CTA's contiguous tile range of a pack; the local
// input vector of each matrix is gathered by xval(local offset) into xs.
template <typename XF>
__device__ void range_phase(Ring& R, int kind, const RangePack& P, double* xs, double* acc, Smem& sm, XF xval) {
  if (R.pre_kind != kind) ring_prefetch(R, kind, P, 0);
  R.pre_kind = 0;
  const long long t0 = P.t_first[blockIdx.x], t1 = P.t_first[blockIdx.x + 1];
  if (t0 >= t1) return;
  const int4 st0 = P.start[blockIdx.x];
  int s = st0.x, I = st0.y, J = st0.z, cur = -1, len = 0, nt = 0;
  for (long long t = t0, k = 0; t < t1; ++t, ++k) {
    if (s != cur) {
      if (cur >= 0) range_flush(P, cur, len, acc);  // same thread owns index i in both loops
      cur = s, nt = P.nt[s], len = kTile * nt;
      const long long xo = P.xoff[s];
      for (int i = threadIdx.x; i < len; i += blockDim.x) xs[i] = xval(xo + i), acc[i] = 0.0;
      __syncthreads();
    }
    const int stg = R.consumed % R.nst;
    mb_wait(&R.full[stg], (R.consumed / R.nst) & 1);
    tile_acc(R.stage + (size_t)stg * kTile * kTile, xs + I * kTile, xs + J * kTile, I == J, acc + I * kTile,
             acc + J * kTile, sm);
    __syncthreads();  // stage consumed, accumulator updated
    if (threadIdx.x == 0) ring_issue(R, P, k + R.nst);
    ++R.consumed;
    if (++J > I) {
      J = 0;
      if (++I == nt) I = 0, ++s;
    }
  }
  range_flush(P, cur, len, acc);
}

// y_s[i] from the partials of the CTAs covering matrix s (CTA order)
__device__ __forceinline__ double range_reduce(const RangePack& P, int s, int i) {
  const int len = kTile * P.nt[s], n = P.ncta[s];
  const double* p = P.part + P.pbase[s] + i;
  double y = 0.0;
  int k = 0;
  for (; k + 4 <= n; k += 4) {
    const double a = __ldcg(p + (long long)k * len), b = __ldcg(p + (long long)(k + 1) * len),
                 c = __ldcg(p + (long long)(k + 2) * len), d = __ldcg(p + (long long)(k + 3) * len);
    y += a, y += b, y += c, y += d;
  }
  for (; k < n; ++k) y += __ldcg(p + (long long)k * len);
  return y;
}

// mode 0: x vector = first ? z : z + beta p (lazy p update); mode 1: x
__device__ void s_tiles_phase(const FusedPcg& A, Ring& R, Smem& sm, double* xs, double* acc, int mode, bool first,
                              double beta) {
  range_phase(R, 1, A.rs, xs, acc, sm, [&](long long o) {
    return mode ? __ldcg(A.li_x + o) : (first ? __ldcg(A.li_z + o) : __ldcg(A.li_z + o) + beta * __ldcg(A.li_p + o));
  });
}

__device__ __forceinline__ double s_reduce(const FusedPcg& A, long long q) {
  const int j = int(q / A.n_iface), gq = int(q % A.n_iface);
  double y = 0.0;
  for (int e = 0; e < A.inv_cnt[gq]; ++e) {
    const int s = A.inv_s[4 * gq + e], pp = A.inv_p[4 * gq + e];
    y += range_reduce(A.rs, s, j * A.ng[s] + pp);
  }
  return y;
}


// z = NN2(r) from the local inputs fr/fc; returns r.z
__device__ double nn2_phases(const FusedPcg& A, Ring& R, Smem& sm, cg::grid_group& g, PhaseClock& pc) {
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x, gstride = (long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const long long gwarp = gtid >> 5, nwarps = gstride >> 5;
  // 4. Psi^T f_r (the first Q tiles stream in meanwhile), Q tiles
  double* xs = dyn_smem + (size_t)A.nst * kTile * kTile;
  ring_prefetch(R, 2, A.rq, A.l2pf);
  auto psi_t = [&]() {
    for (long long wv = gwarp; wv < A.ncol_total; wv += nwarps) {
      int lo = 0, hi = A.NS;  // subdomain s with coff[s] <= wv < coff[s+1]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (A.coff[mid] <= wv) lo = mid; else hi = mid;
      }
      const int s = lo;
      const int c = int(wv - A.coff[s]), rs = A.NT * A.nr[s];
      const double* col = A.Psi + A.psioff[s] + (long long)c * rs;
      const double* f = A.fr + A.roff[s];
      double acc = 0.0;
#pragma unroll kUnroll
      for (int a = lane; a < rs; a += 32) acc += col[a] * f[a];
      acc = warp_sum(acc);
      if (lane == 0) A.dsub[wv] = A.fc[wv] - acc;
    }
  };
  if (A.NC > 0 && !A.psi_late) psi_t();
  range_phase(R, 2, A.rq, xs, xs + A.maxlen, sm, [&](long long o) { return __ldcg(A.fr + o); });
  ring_prefetch(R, 1, A.rs, A.l2pf);  // next iteration's S tiles stream in during 5-7
  if (A.NC > 0 && A.psi_late) psi_t();
  g.sync();
  pc.tick(3);
  if (A.NC > 0) {
    // 5. d = sum_s B_s^T d_s (ascending s)
    for (long long qc = gtid; qc < A.NC; qc += gstride) {
      const int j = int(qc / A.n_corner), gc = int(qc % A.n_corner);
      double d = 0.0;
      for (int e = 0; e < A.cinv_cnt[gc]; ++e) {
        const int s = A.cinv_s[4 * gc + e];
        d += A.dsub[A.coff[s] + (long long)j * A.nc[s] + A.cinv_c[4 * gc + e]];
      }
      A.dco[qc] = d;
    }
    g.sync();
    pc.tick(4);
    // 6. u_c = F_cc^-1 d (symmetric: row = column), plus the per-subdomain
    //    corner copies B_s u_c (c-space, compact)
    for (long long row = gwarp; row < A.NC; row += nwarps) {
      const double* col = A.Finv + row * A.NC;
      double acc = 0.0;
#pragma unroll kUnroll
      for (int c = lane; c < A.NC; c += 32) acc += col[c] * __ldcg(A.dco + c);
      acc = warp_sum(acc);
      if (lane == 0) {
        A.uco[row] = acc;
        const int j = int(row / A.n_corner), gc = int(row % A.n_corner);
        for (int e = 0; e < A.cinv_cnt[gc]; ++e) {
          const int s = A.cinv_s[4 * gc + e];
          A.ucl[A.coff[s] + (long long)j * A.nc[s] + A.cinv_c[4 * gc + e]] = acc;
        }
      }
    }
    g.sync();
    pc.tick(5);
    // 6b. w_s = Psi_s (B_s u_c) on the remaining dofs (r-space, coalesced over rows)
    for (long long i = gtid; i < A.rlen; i += gstride) {
      int lo = 0, hi = A.NS;  // subdomain of padded r-space index i
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (A.roff[mid] <= i) lo = mid; else hi = mid;
      }
      const int s = lo, a = int(i - A.roff[s]), rs = A.NT * A.nr[s];
      if (a >= rs) continue;
      const double* P = A.Psi + A.psioff[s] + a;
      const double* u = A.ucl + A.coff[s];
      const int cs = A.NT * A.nc[s];
      double acc = 0.0;
#pragma unroll kUnroll
      for (int c = 0; c < cs; ++c) acc += P[(long long)c * rs] * __ldcg(u + c);
      A.wr[i] = acc;
    }
    g.sync();
    pc.tick(5);
  }
  // 7. z = sum_s R_s^T D_s zeta_s ; r.z
  double acc = 0.0;
  for (long long q = gtid; q < A.NG; q += gstride) {
    const int j = int(q / A.n_iface), gq = int(q % A.n_iface);
    double zq = 0.0;
    for (int e = 0; e < A.inv_cnt[gq]; ++e) {
      const int s = A.inv_s[4 * gq + e], pp = A.inv_p[4 * gq + e];
      const int kind = A.pkind[A.ip_off[s] + pp];
      const double wgt = A.iface_w[A.ip_off[s] + pp];
      double v;
      if (kind >= 0) {
        const int ar = j * A.nr[s] + kind;
        v = range_reduce(A.rq, s, ar);
        if (A.NC > 0) v -= __ldcg(A.wr + A.roff[s] + ar);  // u_r = Q f_r - Psi u_c
      } else {
        v = A.NC > 0 ? __ldcg(A.ucl + A.coff[s] + (long long)j * A.nc[s] + (-1 - kind)) : 0.0;
      }
      zq += wgt * v;
    }
    A.z[q] = zq;
    write_local_s(A, A.li_z, q, zq);
    acc += A.r[q] * zq;
  }
  const double rzv = grid_sum(acc, A.part, 4, g, sm);
  pc.tick(6);
  return rzv;
}

__global__ void __launch_bounds__(256) pcg_fused_kernel(FusedPcg A) {
  cg::grid_group g = cg::this_grid();
  __shared__ Smem sm;
  __shared__ unsigned long long ring_bar[kMaxRing];
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x, gstride = (long long)gridDim.x * blockDim.x;
  const bool leader = gtid == 0;
  Ring R{dyn_smem, ring_bar, A.nst, 0, 0, 0};
  double* xs = dyn_smem + (size_t)A.nst * kTile * kTile;  // local input vector, then the accumulator
  double* xacc = xs + A.maxlen;
  PhaseClock pc{leader && A.tphase != nullptr, 0, {0, 0, 0, 0, 0, 0, 0, 0}};
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pc.last));
  if (threadIdx.x == 0) {
    for (int i = 0; i < A.nst; ++i) mb_init(&ring_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // x = 0, r = b, NN2 inputs of r, ||b||^2
  double acc = 0.0;
  for (long long q = gtid; q < A.NG; q += gstride) {
    const double bv = A.b[q];
    A.x[q] = 0.0;
    A.r[q] = bv;
    acc += bv * bv;
    write_local(A, q, bv);
  }
  const double bnorm = sqrt(grid_sum(acc, A.part, 0, g, sm));
  int hl = 0;
  if (bnorm == 0.0) {
    if (leader) A.out[0] = 0, A.out[1] = 1, A.out[2] = 1, A.hist[0] = 0.0;
    return;
  }
  if (leader) A.hist[hl] = 1.0;
  ++hl;
  pc.tick(7);
  double rz = nn2_phases(A, R, sm, g, pc);
  double beta = 0.0;
  bool first = true, converged = false;
  int it = 0;
  while (it < A.max_iter) {
    // 1-2: q = S p_new, p.q
    s_tiles_phase(A, R, sm, xs, xacc, 0, first, beta);
    g.sync();
    pc.tick(0);
    acc = 0.0;
    for (long long q = gtid; q < A.NG; q += gstride) {
      const double y = s_reduce(A, q);
      A.q[q] = y;
      acc += y * (first ? A.z[q] : A.z[q] + beta * A.p[q]);
    }
    const double alpha = rz / grid_sum(acc, A.part, 1, g, sm);
    pc.tick(1);
    // 3: p, x, r updates and NN2 inputs
    acc = 0.0;
    for (long long q = gtid; q < A.NG; q += gstride) {
      const double pn = first ? A.z[q] : A.z[q] + beta * A.p[q];
      A.p[q] = pn;
      write_local_s(A, A.li_p, q, pn);
      A.x[q] += alpha * pn;
      const double rn = A.r[q] - alpha * A.q[q];
      A.r[q] = rn;
      acc += rn * rn;
      write_local(A, q, rn);
    }
    const double rr = grid_sum(acc, A.part, 2, g, sm);
    pc.tick(2);
    first = false;
    ++it;
    double rel = sqrt(rr) / bnorm;
    if (rel <= A.tol) {
      // recurrence hit the target; confirm with the true residual b - S x
      for (long long q = gtid; q < A.NG; q += gstride) write_local_s(A, A.li_x, q, A.x[q]);
      g.sync();
      s_tiles_phase(A, R, sm, xs, xacc, 1, false, 0.0);
      g.sync();
      acc = 0.0;
      for (long long q = gtid; q < A.NG; q += gstride) {
        const double rt = A.b[q] - s_reduce(A, q);
        A.q[q] = rt;
        acc += rt * rt;
      }
      rel = sqrt(grid_sum(acc, A.part, 3, g, sm)) / bnorm;
      if (leader && hl < A.hist_cap) A.hist[hl] = rel;
      ++hl;
      if (rel <= A.tol) {
        converged = true;
        break;
      }
      for (long long q = gtid; q < A.NG; q += gstride) {  // restart from r_true, p kept
        const double rt = A.q[q];
        A.r[q] = rt;
        write_local(A, q, rt);
      }
      g.sync();
    } else {
      if (leader && hl < A.hist_cap) A.hist[hl] = rel;
      ++hl;
    }
    pc.tick(7);
    const double rz_next = nn2_phases(A, R, sm, g, pc);
    beta = rz_next / rz;
    rz = rz_next;
  }
  pc.tick(7);
  if (leader) {
    A.out[0] = it;
    A.out[1] = converged ? 1 : 0;
    A.out[2] = hl;
    if (pc.on)
      for (int i = 0; i < 8; ++i) A.tphase[i] += pc.acc[i];
  }
  // drain tile copies still in flight before the CTA's shared memory goes away
  if (threadIdx.x == 0)
    for (int c = R.consumed; c < R.issued; ++c) mb_wait(&R.full[c % R.nst], (c / R.nst) & 1);
  __syncthreads();
}

// --------------------------------------------------------------- host ----
void RangeBufs::plan(const TilePack& tp, int grid) {
  std::vector<long long> tf(grid + 1), pb(tp.nmat + 1, 0);
  std::vector<int4> st(grid, make_int4(0, 0, 0, 0));
  std::vector<int> c0(tp.nmat, 0), nc(tp.nmat, 0);
  for (int c = 0; c <= grid; ++c) tf[c] = tp.n_tiles * c / grid;
  // matrix, I, J of every CTA's first tile; CTAs covering each matrix
  auto cta_of = [&](long long t) {  // CTA whose range holds tile t
    return int(std::upper_bound(tf.begin(), tf.end(), t) - tf.begin()) - 1;
  };
  for (int c = 0; c < grid; ++c) {
    if (tf[c] >= tf[c + 1]) continue;
    const int s = int(std::upper_bound(tp.tile_base.begin(), tp.tile_base.end(), tf[c]) - tp.tile_base.begin()) - 1;
    long long r = tf[c] - tp.tile_base[s];
    int I = 0;
    while (r > I) r -= ++I;  // row-major lower order: row I holds I + 1 tiles
    st[c] = make_int4(s, I, int(r), 0);
  }
  for (int s = 0; s < tp.nmat; ++s) {
    const int a = cta_of(tp.tile_base[s]), b = cta_of(tp.tile_base[s + 1] - 1);
    c0[s] = a, nc[s] = b - a + 1;
    pb[s + 1] = pb[s] + (long long)nc[s] * kTile * tp.ntile[s];
  }
  t_first.upload(tf), start.upload(st);
  this->c0.upload(c0), ncta.upload(nc), pbase.upload(pb);
  part.alloc(std::max<long long>(1, pb[tp.nmat]));
  SGW_CUDA(cudaMemset(part.p, 0, part.n * sizeof(double)));  // slots of CTAs with empty ranges stay 0
}


void GpuSolver::setup_fused_pcg() {
  tphase_.alloc(8), tphase_.zero(st_);
  if (comm_) {  // sharded: the host-driven loop with a sum over ranks after each scatter
    use_fused_ = false;
    return;
  }
  // S-space local gather map (padded like Sp): global flat interface index or -1
  std::vector<int> smap(Sp.xlen, -1);
  for (int s = 0; s < NS; ++s) {
    const auto& sd = G.sub[s];
    for (int j = 0; j < NT; ++j)
      for (int p = 0; p < ng_[s]; ++p) smap[Sp.xoff[s] + (long long)j * ng_[s] + p] = j * G.n_iface + sd.iface_pos[p];
  }
  smap_.upload(smap);
  int dev = 0, sms = 0, nb = 0, smem_sm = 0, smem_blk = 0;
  SGW_CUDA(cudaGetDevice(&dev));
  SGW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SGW_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  SGW_CUDA(cudaDeviceGetAttribute(&smem_blk, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // shared memory per CTA: the tile ring, the local input vector and the
  // accumulator of the longest local vector.  Default two CTAs per SM (more
  // warps for the scatter phases; measured 0.56 vs 0.64 ms per C2 iteration
  // with one CTA and a deeper ring) if each gets >= 2 stages, else one with the
  // deepest ring that fits.  SGW_PCG_BPS / SGW_PCG_RING tune.
  fused_maxlen_ = 0;
  for (int s = 0; s < NS; ++s) fused_maxlen_ = std::max({fused_maxlen_, kTile * Sp.ntile[s], kTile * Qp.ntile[s]});
  cudaFuncAttributes fa{};
  SGW_CUDA(cudaFuncGetAttributes(&fa, (const void*)pcg_fused_kernel));
  int bps = 2;
  if (const char* e = std::getenv("SGW_PCG_BPS")) bps = std::max(1, std::atoi(e));
  const long long vec = 2LL * fused_maxlen_ * 8;
  for (;; --bps) {
    const long long avail = std::min<long long>(smem_blk, smem_sm / bps - 1024) - (long long)fa.sharedSizeBytes - vec;
    fused_nst_ = (int)std::min<long long>(kMaxRing, avail / kTileBytes);
    if (fused_nst_ >= 2 || bps == 1) break;
  }
  if (const char* e = std::getenv("SGW_PCG_RING")) fused_nst_ = std::min(kMaxRing, std::atoi(e));
  if (fused_nst_ < 1) throw Error(4, "persistent PCG: local vectors exceed shared memory");
  fused_smem_ = (size_t)fused_nst_ * kTileBytes + (size_t)vec;
  SGW_CUDA(cudaFuncSetAttribute((const void*)pcg_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)fused_smem_));
  SGW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pcg_fused_kernel, 256, fused_smem_));
  fused_grid_ = std::max(1, std::min(nb, bps)) * sms;
  rs_.plan(Sp, fused_grid_);
  rq_.plan(Qp, fused_grid_);
  fused_part_.alloc(size_t(8) * fused_grid_);
  fused_out_.alloc(4);
  fused_hist_.alloc(P.max_iter + 8);
  for (DBuf<double>* b : {&li_z_, &li_p_, &li_xx_}) b->alloc(Sp.xlen), b->zero(st_);  // padding stays 0
  ucl_.alloc(std::max<long long>(1, coff_.back())), ucl_.zero(st_);
  wr_.alloc(std::max<long long>(1, Qp.xlen)), wr_.zero(st_);
  const char* e = std::getenv("SGW_PCG");
  use_fused_ = !(e && std::string(e) == "host");
}

int GpuSolver::pcg_fused(const double* b, double* x, bool* converged, std::vector<double>* hist) {
  cudaEventRecord(ev_[0], st_);
  FusedPcg A{};
  A.NG = NG;
  A.ncol_total = coff_.back();
  A.n_iface = G.n_iface, A.NT = NT, A.NS = NS, A.n_corner = G.n_corner, A.NC = NC;
  A.max_iter = P.max_iter, A.hist_cap = (int)fused_hist_.n, A.tol = P.tol;
  A.b = b, A.x = x, A.r = vr.p, A.z = vz.p, A.p = vp.p, A.q = vq.p;
  A.s_desc = Sp.desc.p, A.s_tiles = Sp.tiles.p, A.s_ntiles = Sp.n_tiles, A.s_row = Sp.rowpart.p,
  A.s_col = Sp.colpart.p, A.s_base = Sp.d_tile_base.p, A.s_xoff = Sp.d_xoff.p, A.s_nt = Sp.d_ntile.p,
  A.smap = smap_.p;
  A.q_desc = Qp.desc.p, A.q_tiles = Qp.tiles.p, A.q_ntiles = Qp.n_tiles, A.q_row = Qp.rowpart.p,
  A.q_col = Qp.colpart.p, A.q_base = Qp.d_tile_base.p, A.q_xoff = Qp.d_xoff.p, A.q_nt = Qp.d_ntile.p;
  A.fr = r_x.p, A.fc = c_f.p;
  A.inv_cnt = inv_cnt.p, A.inv_s = inv_s.p, A.inv_p = inv_p.p, A.ip_off = ip_off.p, A.ng = ng_d.p, A.nr = nr_d.p,
  A.nc = nc_d.p, A.pkind = pkind_.p, A.cpos_flat = cpos_flat_.p, A.cp_off = cp_off_.p, A.iface_w = iface_w.p;
  A.cinv_cnt = cinv_cnt.p, A.cinv_s = cinv_s.p, A.cinv_c = cinv_c.p;
  A.roff = d_roff.p, A.coff = d_coff.p, A.psioff = d_psioff.p;
  A.Psi = Psi.p, A.Finv = Finv.p, A.dsub = c_d.p, A.dco = dcoarse.p, A.uco = ucoarse.p;
  A.part = fused_part_.p, A.out = fused_out_.p, A.hist = fused_hist_.p;
  A.s_tx = Sp.tx.p, A.q_tx = Qp.tx.p;
  A.li_z = li_z_.p, A.li_p = li_p_.p, A.li_x = li_xx_.p;
  A.tphase = KP.on ? tphase_.p : nullptr;
  A.ucl = ucl_.p, A.wr = wr_.p, A.rlen = Qp.xlen;
  A.rs = RangePack{Sp.tiles.p, Sp.d_ntile.p, Sp.d_xoff.p, rs_.t_first.p, rs_.start.p, rs_.c0.p, rs_.ncta.p, rs_.pbase.p, rs_.part.p};
  A.rq = RangePack{Qp.tiles.p, Qp.d_ntile.p, Qp.d_xoff.p, rq_.t_first.p, rq_.start.p, rq_.c0.p, rq_.ncta.p, rq_.pbase.p, rq_.part.p};
  A.nst = fused_nst_, A.maxlen = fused_maxlen_;
  A.l2pf = 0, A.psi_late = 1;
  if (const char* e = std::getenv("SGW_PCG_PSI_LATE")) A.psi_late = std::atoi(e);  // tuning hook
  if (const char* e = std::getenv("SGW_PCG_L2PF")) A.l2pf = std::max(0, std::atoi(e));  // tuning hook
  void* args[] = {&A};
  SGW_CUDA(cudaLaunchCooperativeKernel((const void*)pcg_fused_kernel, dim3(fused_grid_), dim3(256), args,
                                       fused_smem_, st_));
  SGW_LAUNCHED();
  int out[3] = {0, 0, 0};
  SGW_CUDA(cudaMemcpyAsync(out, fused_out_.p, sizeof(out), cudaMemcpyDeviceToHost, st_));
  cudaEventRecord(ev_[1], st_);
  SGW_CUDA(cudaEventSynchronize(ev_[1]));
  float ms = 0;
  cudaEventElapsedTime(&ms, ev_[0], ev_[1]);
  T.pcg_ms += ms;
  T.iterations += out[0];
  T.matvecs += out[0];
  T.nn2s += out[0];
  *converged = out[1] != 0;
  const int hl = std::min<int>(out[2], (int)fused_hist_.n);
  std::vector<double> h(std::max(hl, 1));
  SGW_CUDA(cudaMemcpy(h.data(), fused_hist_.p, hl * sizeof(double), cudaMemcpyDeviceToHost));
  last_rel = hl > 0 ? h[hl - 1] : 0.0;
  if (hist) {
    h.resize(hl);
    *hist = h;
  }
  return out[0];
}

}  // namespace sgw
