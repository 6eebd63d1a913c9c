// The whole interface PCG solve (src/pcg.cpp:7-50) with the NN2 preconditioner
// (src/dd.cpp:199-253) as ONE persistent cooperative kernel: every CTA walks
// the same phase sequence separated by grid barriers, so a PCG iteration costs
// eight grid barriers instead of a dozen launches plus a host round trip for
// the convergence test.
//
// Per iteration (phase -> grid barrier):
//   1. S walk       the CTA's contiguous range of S_s tiles on p_new = z + beta p
//                   (local vectors and accumulators in shared memory)
//   2. S scatter    q = sum_s R_s^T S_s R_s p_new from the CTA partials, p.q
//   3. update       p = p_new, x += alpha p, r -= alpha q, r.r, and the
//                   weighted local copies D_s R_s r (NN2 inputs f_r, f_c)
//   4. Q / Psi walk Q_s f_r and Psi_s^T f_r (Psi as rectangular tiles)
//   5. coarse       d = sum_s B_s^T (f_c - Psi_s^T f_r)
//   6. coarse solve u_c = F_cc^-1 d; Psi walk on B_s u_c
//   7. z scatter    z = sum_s R_s^T D_s [Q f_r - Psi u_c ; u_c], r.z
// Every tile stream goes through a per-CTA TMA ring (evict-first); a walk
// issues the next walk's first tiles during its tail.  Reductions: fixed-order
// block sums, then every CTA sums the block partials in index order itself
// (bitwise identical in every CTA, run to run).  The convergence test, the
// true-residual confirmation and the restart from the true residual are
// evaluated on device exactly as src/pcg.cpp:30-40.
#include <cooperative_groups.h>
#include <cstdio>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "solver.cuh"
#include "tiles.cuh"

namespace cg = cooperative_groups;

namespace sgw {

struct FusedPcg {
  long long NG;
  int n_iface, NT, NS, n_corner, NC, max_iter, hist_cap;
  double tol;
  const double* b;
  double *x, *r, *z, *p;
  double* q;                     // scratch (true residual)
  const long long *s_xoff, *q_xoff;
  double *fr, *fc;
  const int *inv_cnt, *inv_s, *inv_p, *ip_off, *ng, *nr, *nc, *pkind;
  const double* iface_w;
  const int *cinv_cnt, *cinv_s, *cinv_c;
  const long long *roff, *coff;
  const double* Finv;
  double *dco, *uco, *ucl;       // d, u_c (flat coarse), B_s u_c (c-space, compact)
  double* part;  // 8 slots x gridDim
  int* out;      // [0] iterations, [1] converged
  double* hist;  // residual history, hist_cap entries
  double *li_z, *li_p, *li_x;    // z, p, x in S-local layout (written by their producers)
  double* tphase;                // 8 accumulated phase times (ns), CTA 0
  RangePack rs, rq, rp;          // contiguous tile ranges per CTA of S, Q and Psi^T
  int nst, maxlen;               // ring stages; longest local vector (doubles)
  // phase-split PCG (sharded runs, pcg_phase_kernel): halo of the shared
  // interface nodes, ownership mask of the dots, the buffer the collectives
  // reduce ([0, NC) coarse d, then XR rr | b.b, XPQ p.q, XRZ r.z, XRT rt.rt)
  // and the device-resident CG state
  HaloDev H;
  const double* own;             // NG, null: every entry owned
  double* xch;
  double* sc;                    // [SC_RZ] r.z, [SC_BNORM] ||b||, [SC_BETA]
  int* st;                       // [ST_IT], [ST_HL], [ST_EXIT], [ST_FIRST], [ST_PFIRST]
  unsigned long long cond;       // conditional handle of the graph's WHILE loop
  int use_cond;
  int l2_keep;                   // tile loads with the default L2 policy (the tile set fits in L2)
  int ph_prefetch;               // phase-split kernels: L2 prefetch of the next walk's first tiles
  // glue descriptors per (interface node gq, slot e): 4 * gq + e (build_scatter_desc)
  const int4* ifd;   // {S-local base (-1: unused slot), S-local term stride, fr / fc base, fr stride (> 0) or -(fc stride)}
  const double* ifw; // partition-of-unity weight of the slot
  const int4* sred;  // S partials {base, term stride, CTA stride, CTAs} (CTAs 0: unused)
  const int4* zred;  // Q partials {base, term stride, CTA stride, CTAs}; CTAs -1: corner (ucl base, stride); -2: unused
  const int4* pred;  // Psi (remaining-dof part) partials {base, term stride, CTA stride, CTAs}
};
enum { SC_RZ = 0, SC_BNORM = 1, SC_BETA = 2 };
enum { ST_IT = 0, ST_HL = 1, ST_EXIT = 2, ST_FIRST = 3, ST_PFIRST = 4 };
// ST_EXIT: 0 running, 1 recurrence residual <= tol (confirm), 2 max_iter,
// 3 b = 0, 4 converged (true residual), 5 true residual failed (restart)
enum { EX_RUN = 0, EX_CHECK = 1, EX_MAXIT = 2, EX_ZERO = 3, EX_CONV = 4, EX_RESTART = 5 };

extern __shared__ __align__(128) double dyn_smem[];  // ring stages, local vector, accumulator

struct Smem {
  double csum[8][kTile];
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
// keep: the whole tile set fits in L2 (small configs such as C1): the default
// policy, so the tiles stay L2-resident across iterations.
__device__ __forceinline__ void mb_load(void* dst, const void* src, unsigned bytes, unsigned long long* b, bool keep) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
  if (keep) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(b))
                 : "memory");
    return;
  }
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
  int keep;              // L2 policy of the tile loads (mb_load)
};

// tile k of this CTA's range of P, continuing into the range of `next` past
// its end (the next walk's first tiles stream in during this one's tail)
__device__ __forceinline__ void ring_issue(Ring& R, const RangePack& P, long long k, const RangePack* next) {
  const RangePack* Q = &P;
  long long t = P.t_first[blockIdx.x] + k;
  const long long t1 = P.t_first[blockIdx.x + 1];
  if (t >= t1) {
    if (!next) return;
    Q = next;
    t = next->t_first[blockIdx.x] + (t - t1);
    if (t >= next->t_first[blockIdx.x + 1]) return;
  }
  const double* src = Q->tiles + (Q->toff ? Q->toff[t] : t * (kTile * kTile));
  const unsigned bytes = Q->tbytes ? (unsigned)Q->tbytes[t] : kTileBytes;
  const int st = R.issued % R.nst;
  mb_load(R.stage + (size_t)st * kTile * kTile, src, bytes, &R.full[st], R.keep != 0);
  ++R.issued;
}
// the first n tiles of this CTA's range of P into L2 (thread 0)
__device__ __forceinline__ void l2_prefetch_range(const RangePack& P, int n) {
  if (threadIdx.x != 0) return;
  const long long t0 = P.t_first[blockIdx.x], t1 = P.t_first[blockIdx.x + 1];
  for (long long t = t0; t < t1 && t < t0 + n; ++t) {
    const double* src = P.tiles + (P.toff ? P.toff[t] : t * (kTile * kTile));
    const unsigned bytes = P.tbytes ? (unsigned)P.tbytes[t] : kTileBytes;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
  }
}

// issue the first tiles of set `kind` for the next tile phase (thread 0).
// The ring always holds the next nst tiles of the consumption sequence: a
// walk of P chained to `next` consumes P's range, then next's; a walk without
// `next` leaves the ring empty.
__device__ __forceinline__ void ring_prefetch(Ring& R, int kind, const RangePack& P, const RangePack* next) {
  if (threadIdx.x == 0)
    for (int n = 0; n < R.nst; ++n) ring_issue(R, P, n, next);
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
#pragma unroll
  for (int e = 0; e < 4; ++e) {  // every slot's descriptor loads at once (unused slots: x < 0)
    const int4 d = __ldg(A.ifd + 4 * gq + e);
    const double wv = __ldg(A.ifw + 4 * gq + e) * val;
    if (d.x >= 0) {
      if (d.w > 0) A.fr[d.z + (long long)j * d.w] = wv;
      else A.fc[d.z - (long long)j * d.w] = wv;
    }
  }
}

// R_s val into an S-local buffer for every subdomain sharing interface index q.
__device__ __forceinline__ void write_local_s(const FusedPcg& A, double* li, long long q, double val) {
  const int j = int(q / A.n_iface), gq = int(q % A.n_iface);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int4 d = __ldg(A.ifd + 4 * gq + e);
    if (d.x >= 0) li[d.x + (long long)j * d.y] = val;
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
// input vector of each matrix s is gathered by xval(s, i) into xs.  With
// `next`, the first tiles of next's range are issued during this walk's tail
// (the caller then marks them as prefetched).
template <typename XF>
__device__ void range_phase(Ring& R, int kind, const RangePack& P, const RangePack* next, double* xs, double* acc,
                            Smem& sm, XF xval) {
  if (R.pre_kind != kind) ring_prefetch(R, kind, P, next);
  R.pre_kind = 0;
  const long long t0 = P.t_first[blockIdx.x], t1 = P.t_first[blockIdx.x + 1];
  if (t0 >= t1) return;
  const int4 st0 = P.start[blockIdx.x];
  int s = st0.x, I = st0.y, J = st0.z, cur = -1, len = 0, nI = 0, nJ = 0, xoJ = 0;
  for (long long t = t0, k = 0; t < t1; ++t, ++k) {
    if (s != cur) {
      if (cur >= 0) range_flush(P, cur, len, acc);  // same thread owns index i in both loops
      cur = s, nI = P.nI[s], nJ = P.rect ? P.nJ[s] : nI;
      xoJ = P.rect ? kTile * nI : 0;
      len = kTile * (P.rect ? nI + nJ : nI);
      for (int i = threadIdx.x; i < len; i += blockDim.x) xs[i] = xval(s, i), acc[i] = 0.0;
      __syncthreads();
    }
    const int stg = R.consumed % R.nst;
    mb_wait(&R.full[stg], (R.consumed / R.nst) & 1);
    tile_acc(R.stage + (size_t)stg * kTile * kTile, xs + I * kTile, xs + xoJ + J * kTile, !P.rect && I == J,
             acc + I * kTile, acc + xoJ + J * kTile, sm);
    __syncthreads();  // stage consumed, accumulator updated
    if (threadIdx.x == 0) ring_issue(R, P, k + R.nst, next);
    ++R.consumed;
    if (P.rect ? ++J == nJ : ++J > I) {
      J = 0;
      if (++I == nI) I = 0, ++s;
    }
  }
  range_flush(P, cur, len, acc);
}

// mode 0: x vector = first ? z : z + beta p (lazy p update); mode 1: x
__device__ void s_tiles_phase(const FusedPcg& A, Ring& R, Smem& sm, double* xs, double* acc, int mode, bool first,
                              double beta) {
  range_phase(R, 1, A.rs, nullptr, xs, acc, sm, [&](int s, int i) {
    const long long o = A.s_xoff[s] + i;
    return mode ? __ldcg(A.li_x + o) : (first ? __ldcg(A.li_z + o) : __ldcg(A.li_z + o) + beta * __ldcg(A.li_p + o));
  });
}

// sum over the sharing subdomains (ascending s) of their S partials at q
__device__ __forceinline__ double s_reduce(const FusedPcg& A, long long q) {
  const int j = int(q / A.n_iface), gq = int(q % A.n_iface);
  int4 d[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) d[e] = __ldg(A.sred + 4 * gq + e);
  // the (<= 4) subdomains' partial lists side by side (tiles.cuh partial_sums)
  const double* p[4];
  int len[4], n[4];
  double ys[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const bool on = d[e].w > 0;
    p[e] = on ? A.rs.part + d[e].x + (long long)j * d[e].y : A.rs.part;
    len[e] = d[e].z, n[e] = on ? d[e].w : 0;
  }
  partial_sums<4, 2>(p, len, n, ys);
  double y = 0.0;
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (d[e].w > 0) y += ys[e];
  return y;
}

// z_q = sum_s w_s [Q_s f_r - Psi_s u_c ; u_c]_q (NN2 step 7), ascending s
__device__ __forceinline__ double z_reduce(const FusedPcg& A, int j, int gq, bool coarse) {
  int4 d[4], p[4];
  double w[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) d[e] = __ldg(A.zred + 4 * gq + e), p[e] = __ldg(A.pred + 4 * gq + e), w[e] = __ldg(A.ifw + 4 * gq + e);
  // lists 0..3: Q_s f_r partials, 4..7: Psi_s u_c partials, all in flight
  // together; corner slots (w == -1) read u_c directly.  The descriptors are
  // folded into pointers / counts / a slot kind before the loads start (the
  // kernel runs two CTAs per SM: 128 registers)
  const double* lp[8];
  int len[8], n[8], kind[4];
  double ys[8], uc[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const bool on = d[e].w >= 0, onp = on && coarse;
    kind[e] = on ? 1 : d[e].w == -1 ? 2 : 0;
    lp[e] = on ? A.rq.part + d[e].x + (long long)j * d[e].y : A.rq.part;
    len[e] = d[e].z, n[e] = on ? d[e].w : 0;
    lp[4 + e] = onp ? A.rp.part + p[e].x + (long long)j * p[e].y : A.rq.part;
    len[4 + e] = p[e].z, n[4 + e] = onp ? p[e].w : 0;
    uc[e] = kind[e] == 2 && coarse ? __ldcg(A.ucl + d[e].x + (long long)j * d[e].y) : 0.0;
  }
  partial_sums<8, 1>(lp, len, n, ys);
  double zq = 0.0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    double v;
    if (kind[e] == 1) {
      v = ys[e];
      if (coarse) v -= ys[4 + e];
    } else if (kind[e] == 2) {
      v = uc[e];
    } else {
      continue;
    }
    zq += w[e] * v;
  }
  return zq;
}


// The persistent kernel's loops over the interface dofs: runs of 32 consecutive
// dofs (one warp reads consecutive entries) dealt round-robin over the CTAs.
// With q = global thread id a small problem (C1: 2,268 dofs) put every dof on
// the first 9 of 148 CTAs, whose load paths then carried all the partial-list
// reads of a scatter phase.  Every loop uses the same map, so a dof stays with
// one thread from loop to loop.
#define FOR_IFACE_DOF(q)                                                                                  \
  for (long long q##_run = (long long)(threadIdx.x >> 5) * gridDim.x + blockIdx.x,                       \
                 q = q##_run * 32 + (threadIdx.x & 31);                                                  \
       q##_run * 32 < A.NG;                                                                              \
       q##_run += (long long)(blockDim.x >> 5) * gridDim.x, q = q##_run * 32 + (threadIdx.x & 31))       \
    if (q < A.NG)

// z = NN2(r) from the local inputs fr/fc; returns r.z.
//  4. Q_s f_r and Psi_s^T f_r: the Q tile walk, then the Psi^T tile walk on
//     [0 | f_r] (corner part of its partials = Psi^T f_r)
//  5. d = sum_s B_s^T (f_c - Psi_s^T f_r) (ascending s)
//  6. u_c = F_cc^-1 d, and B_s u_c per subdomain (c-space)
//  6b. Psi_s B_s u_c: the Psi^T tile walk on [B_s u_c | 0] (remaining-dof part)
//  7. z = sum_s R_s^T D_s [Q f_r - Psi u_c ; u_c], r.z
// Psi is read twice per iteration, as the reference's two S_rc products.
__device__ double nn2_phases(const FusedPcg& A, Ring& R, Smem& sm, cg::grid_group& g, PhaseClock& pc) {
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x, gstride = (long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const long long gwarp = gtid >> 5, nwarps = gstride >> 5;
  double* xs = dyn_smem + (size_t)A.nst * kTile * kTile;
  double* acc = xs + A.maxlen;
  const bool coarse = A.NC > 0;
  // 4.
  range_phase(R, 2, A.rq, coarse ? &A.rp : &A.rs, xs, acc, sm,
              [&](int s, int i) { return __ldcg(A.fr + A.q_xoff[s] + i); });
  if (coarse) {
    R.pre_kind = 3;
    range_phase(R, 3, A.rp, nullptr, xs, acc, sm, [&](int s, int i) {
      const int o = i - kTile * A.rp.nI[s];  // remaining-dof part: f_r (padded r-space layout)
      return o >= 0 ? __ldcg(A.fr + A.roff[s] + o) : 0.0;
    });
    // the ring is empty: the same tiles again for 6b (then the next
    // iteration's S tiles) stream in during 5-6
    ring_prefetch(R, 3, A.rp, &A.rs);
  } else {
    R.pre_kind = 1;  // next iteration's S tiles stream in during 7
  }
  g.sync();
  pc.tick(3);
  if (coarse) {
    // 5. one warp per coarse dof: lane group e (8 lanes) takes subdomain e
    //    (<= 4 share a cross point), its lanes split the CTA partials
    for (long long qc = blockIdx.x + (long long)(threadIdx.x >> 5) * gridDim.x; qc < A.NC; qc += nwarps) {
      const int j = int(qc / A.n_corner), gc = int(qc % A.n_corner), e = lane >> 3, kk = lane & 7;
      double d = 0.0;
      if (e < A.cinv_cnt[gc]) {
        const int s = A.cinv_s[4 * gc + e], c = j * A.nc[s] + A.cinv_c[4 * gc + e];
        const int len = kTile * (A.rp.nI[s] + A.rp.nJ[s]), n = A.rp.ncta[s];
        const double* pp = A.rp.part + A.rp.pbase[s] + c;
        for (int k = kk; k < n; k += 8) d -= __ldcg(pp + (long long)k * len);
        if (kk == 0) d += __ldcg(A.fc + A.coff[s] + c);
      }
      d = warp_sum(d);
      if (lane == 0) A.dco[qc] = d;
    }
    g.sync();
    pc.tick(4);
    // 6. (F_cc^-1 symmetric: row = column).  d staged in shared memory when
    //    it fits; rows streamed with 16-byte loads
    const bool dsm = A.NC <= 2 * A.maxlen;
    if (dsm) {
      for (int c = threadIdx.x; c < A.NC; c += blockDim.x) xs[c] = __ldcg(A.dco + c);
      __syncthreads();
    }
    // rows dealt round-robin over the CTAs first (row = b + (warp + 8 i) G):
    // every SM streams its share of F_cc^-1 even when n_C < number of warps
    const int nw = blockDim.x >> 5;
    for (long long row = blockIdx.x + (long long)(threadIdx.x >> 5) * gridDim.x; row < A.NC;
         row += (long long)nw * gridDim.x) {
      const double* col = A.Finv + row * A.NC;
      auto dv = [&](int c) { return dsm ? xs[c] : __ldcg(A.dco + c); };
      const int h = int((row * A.NC) & 1);  // leading element before the 16-byte aligned part
      const int n2 = (A.NC - h) >> 1;
      const double2* c2 = reinterpret_cast<const double2*>(col + h);
      double a = 0.0;
#pragma unroll kUnroll
      for (int k = lane; k < n2; k += 32) {
        const double2 v = __ldg(c2 + k);
        a += v.x * dv(h + 2 * k) + v.y * dv(h + 2 * k + 1);
      }
      if (lane == 0) {
        if (h) a += __ldg(col) * dv(0);
        if ((A.NC - h) & 1) a += __ldg(col + A.NC - 1) * dv(A.NC - 1);
      }
      a = warp_sum(a);
      if (lane == 0) {
        A.uco[row] = a;
        const int j = int(row / A.n_corner), gc = int(row % A.n_corner);
        for (int e = 0; e < A.cinv_cnt[gc]; ++e) {
          const int s = A.cinv_s[4 * gc + e];
          A.ucl[A.coff[s] + (long long)j * A.nc[s] + A.cinv_c[4 * gc + e]] = a;
        }
      }
    }
    g.sync();
    pc.tick(5);
    // 6b.
    range_phase(R, 3, A.rp, &A.rs, xs, acc, sm, [&](int s, int i) {
      return i < A.NT * A.nc[s] ? __ldcg(A.ucl + A.coff[s] + i) : 0.0;
    });
    R.pre_kind = 1;  // next iteration's S tiles stream in during 7
    g.sync();
    pc.tick(5);
  }
  // 7.
  double rz = 0.0;
  FOR_IFACE_DOF(q) {
    const int j = int(q / A.n_iface), gq = int(q % A.n_iface);
    const double zq = z_reduce(A, j, gq, coarse);  // u_r = Q f_r - Psi u_c ; u_c
    A.z[q] = zq;
    write_local_s(A, A.li_z, q, zq);
    rz += A.r[q] * zq;
  }
  const double rzv = grid_sum(rz, A.part, 4, g, sm);
  pc.tick(6);
  return rzv;
}

__global__ void __launch_bounds__(256, 2) pcg_fused_kernel(FusedPcg A) {
  cg::grid_group g = cg::this_grid();
  __shared__ Smem sm;
  __shared__ unsigned long long ring_bar[kMaxRing];
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x, gstride = (long long)gridDim.x * blockDim.x;
  const bool leader = gtid == 0;
  Ring R{dyn_smem, ring_bar, A.nst, 0, 0, 0, A.l2_keep};
  double* xs = dyn_smem + (size_t)A.nst * kTile * kTile;  // local input vector, then the accumulator
  double* xacc = xs + A.maxlen;
  PhaseClock pc{leader && A.tphase != nullptr, 0, {0, 0, 0, 0, 0, 0, 0, 0}};
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pc.last));
  // stages start zeroed: rows past a narrow Psi chunk then always hold finite
  // values (they only meet zero inputs or padding outputs)
  for (int i = threadIdx.x; i < A.nst * kTile * kTile; i += blockDim.x) dyn_smem[i] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the first bulk copy overwrites them
  if (threadIdx.x == 0) {
    for (int i = 0; i < A.nst; ++i) mb_init(&ring_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // x = 0, r = b, NN2 inputs of r, ||b||^2
  double acc = 0.0;
  FOR_IFACE_DOF(q) {
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
    FOR_IFACE_DOF(q) {
      const double y = s_reduce(A, q);
      A.q[q] = y;
      acc += y * (first ? A.z[q] : A.z[q] + beta * A.p[q]);
    }
    const double alpha = rz / grid_sum(acc, A.part, 1, g, sm);
    pc.tick(1);
    // 3: p, x, r updates and NN2 inputs
    acc = 0.0;
    FOR_IFACE_DOF(q) {
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
      FOR_IFACE_DOF(q) write_local_s(A, A.li_x, q, A.x[q]);
      g.sync();
      s_tiles_phase(A, R, sm, xs, xacc, 1, false, 0.0);
      g.sync();
      acc = 0.0;
      FOR_IFACE_DOF(q) {
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
      FOR_IFACE_DOF(q) {  // restart from r_true, p kept
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

// One tile walk as a standalone (non-cooperative) launch, for the host-driven
// PCG of sharded runs: every CTA walks its range of P on the local vector x
// (layout xoff) and writes its partials; consumers use range_reduce.
__global__ void __launch_bounds__(256) walk_kernel(RangePack P, const double* __restrict__ x,
                                                   const long long* __restrict__ xoff, int nst, int maxlen,
                                                   int xmode, const int* __restrict__ ncs) {
  __shared__ Smem sm;
  __shared__ unsigned long long ring_bar[kMaxRing];
  Ring R{dyn_smem, ring_bar, nst, 0, 0, 0};
  double* xs = dyn_smem + (size_t)nst * kTile * kTile;
  for (int i = threadIdx.x; i < nst * kTile * kTile; i += blockDim.x) dyn_smem[i] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) mb_init(&ring_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // xmode 0: x[xoff[s] + i]; Psi^T tiles: 1 = [0 | f_r] (xoff = r-space offsets),
  // 2 = [B_s u_c | 0] (xoff = c-space offsets, ncs = corner columns per matrix)
  range_phase(R, 1, P, nullptr, xs, xs + maxlen, sm, [&](int s, int i) {
    if (xmode == 0) return __ldg(x + xoff[s] + i);
    const int o = i - kTile * P.nI[s];
    if (xmode == 1) return o >= 0 ? __ldcg(x + xoff[s] + o) : 0.0;
    return i < ncs[s] ? __ldcg(x + xoff[s] + i) : 0.0;
  });
  if (threadIdx.x == 0)
    for (int c = R.consumed; c < R.issued; ++c) mb_wait(&R.full[c % R.nst], (c / R.nst) & 1);
  __syncthreads();
}

// ------------------------------------------------- phase-split PCG -------
// The persistent kernel's iteration cut at its cross-rank sums, for sharded
// runs.  One iteration = four cooperative launches with the
// exchanges between them (captured with them in one CUDA graph whose WHILE
// conditional node keeps the convergence test on the device):
//   A  combine z's shared nodes; beta; q_partial = sum_{s owned} R_s^T S_s R_s p
//      (tile walk + scatter), p.q partial, pack q      -> halo(q), allreduce(p.q)
//   B  combine q; alpha; p, x, r updates; r.r partial (owned nodes)
//                                                      -> allreduce(r.r)
//   B2 convergence test (loop condition); unless it ends the loop, NN2 up to
//      the coarse partial d                            -> allreduce(d)
//   C  u_c = F_cc^-1 d; Psi u_c; z partial, r.z partial, pack z
//                                                      -> halo(z), allreduce(r.z)
// The test precedes NN2 as in src/pcg.cpp:30-44: the converged iteration
// streams no Q / Psi tiles (a fused B + B2 did, one wasted NN2 per solve).
// p.q and r.z are sums of per-subdomain dots (p.q = sum_s (R_s p).(S_s R_s p),
// r.z = sum_s (R_s r).(D_s zeta_s)), so their partials need no halo.
enum { PH_INIT = 0, PH_C0, PH_A, PH_B, PH_C, PH_T1, PH_T2, PH_R, PH_RC0, PH_B2 };

__device__ __forceinline__ bool owned(const FusedPcg& A, long long q) { return !A.own || A.own[q] != 0.0; }

// Q_s f_r, Psi_s^T f_r tile walks, then the coarse partial d -> xch[0, NC)
__device__ void ph_nn2a(const FusedPcg& A, Ring& R, Smem& sm, cg::grid_group& g, double* xs, double* acc) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * blockDim.x >> 5;
  const bool coarse = A.NC > 0;
  range_phase(R, 2, A.rq, coarse ? &A.rp : nullptr, xs, acc, sm,
              [&](int s, int i) { return __ldcg(A.fr + A.q_xoff[s] + i); });
  if (coarse) {
    R.pre_kind = 3;
    range_phase(R, 3, A.rp, nullptr, xs, acc, sm, [&](int s, int i) {
      const int o = i - kTile * A.rp.nI[s];
      return o >= 0 ? __ldcg(A.fr + A.roff[s] + o) : 0.0;
    });
  }
  g.sync();
  if (!coarse) return;
  for (long long qc = blockIdx.x + (long long)(threadIdx.x >> 5) * gridDim.x; qc < A.NC; qc += nwarps) {
    const int j = int(qc / A.n_corner), gc = int(qc % A.n_corner), e = lane >> 3, kk = lane & 7;
    double d = 0.0;
    if (e < A.cinv_cnt[gc]) {
      const int s = A.cinv_s[4 * gc + e], c = j * A.nc[s] + A.cinv_c[4 * gc + e];
      const int len = kTile * (A.rp.nI[s] + A.rp.nJ[s]), n = A.rp.ncta[s];
      const double* pp = A.rp.part + A.rp.pbase[s] + c;
      for (int k = kk; k < n; k += 8) d -= __ldcg(pp + (long long)k * len);
      if (kk == 0) d += __ldcg(A.fc + A.coff[s] + c);
    }
    d = warp_sum(d);
    if (lane == 0) A.xch[qc] = d;  // this rank's partial of B^T d
  }
}

// u_c = F_cc^-1 d (d summed over ranks in xch), Psi_s B_s u_c, then the local
// partial z = sum_{s owned} R_s^T D_s zeta_s (packed for the halo); returns the
// grid total of the partial r.z (valid in every thread)
__device__ double ph_nn2b(const FusedPcg& A, Ring& R, Smem& sm, cg::grid_group& g, double* xs, double* acc) {
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x, gstride = (long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const bool coarse = A.NC > 0;
  if (coarse) {
    const bool dsm = A.NC <= 2 * A.maxlen;
    if (dsm) {
      for (int c = threadIdx.x; c < A.NC; c += blockDim.x) xs[c] = __ldcg(A.xch + c);
      __syncthreads();
    }
    const int nw = blockDim.x >> 5;
    for (long long row = blockIdx.x + (long long)(threadIdx.x >> 5) * gridDim.x; row < A.NC;
         row += (long long)nw * gridDim.x) {
      const double* col = A.Finv + row * A.NC;
      auto dv = [&](int c) { return dsm ? xs[c] : __ldcg(A.xch + c); };
      const int h = int((row * A.NC) & 1);
      const int n2 = (A.NC - h) >> 1;
      const double2* c2 = reinterpret_cast<const double2*>(col + h);
      double a = 0.0;
#pragma unroll kUnroll
      for (int k = lane; k < n2; k += 32) {
        const double2 v = __ldg(c2 + k);
        a += v.x * dv(h + 2 * k) + v.y * dv(h + 2 * k + 1);
      }
      if (lane == 0) {
        if (h) a += __ldg(col) * dv(0);
        if ((A.NC - h) & 1) a += __ldg(col + A.NC - 1) * dv(A.NC - 1);
      }
      a = warp_sum(a);
      if (lane == 0) {
        A.uco[row] = a;
        const int j = int(row / A.n_corner), gc = int(row % A.n_corner);
        for (int e = 0; e < A.cinv_cnt[gc]; ++e) {
          const int s = A.cinv_s[4 * gc + e];
          A.ucl[A.coff[s] + (long long)j * A.nc[s] + A.cinv_c[4 * gc + e]] = a;
        }
      }
    }
    g.sync();
    range_phase(R, 3, A.rp, nullptr, xs, acc, sm, [&](int s, int i) {
      return i < A.NT * A.nc[s] ? __ldcg(A.ucl + A.coff[s] + i) : 0.0;
    });
    g.sync();
  }
  double rz = 0.0;
  for (long long q = gtid; q < A.NG; q += gstride) {
    const int j = int(q / A.n_iface), gq = int(q % A.n_iface);
    const double zq = z_reduce(A, j, gq, coarse);
    A.z[q] = zq;
    write_local_s(A, A.li_z, q, zq);  // shared nodes are rewritten after their halo
    halo_pack_one(A.H, j, gq, zq);
    rz += A.r[q] * zq;
  }
  return grid_sum(rz, A.part, 4, g, sm);
}

__global__ void __launch_bounds__(256) pcg_phase_kernel(FusedPcg A, int which) {
  cg::grid_group g = cg::this_grid();
  __shared__ Smem sm;
  __shared__ unsigned long long ring_bar[kMaxRing];
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x, gstride = (long long)gridDim.x * blockDim.x;
  const bool leader = gtid == 0;
  Ring R{dyn_smem, ring_bar, A.nst, 0, 0, 0, A.l2_keep};
  double* xs = dyn_smem + (size_t)A.nst * kTile * kTile;
  double* xacc = xs + A.maxlen;
  // only the phases that walk Psi's narrow tiles need zeroed stages (rows past
  // a narrow chunk must hold finite values); PH_B walks no tiles at all
  const bool walks_psi = which == PH_INIT || which == PH_C0 || which == PH_B2 || which == PH_C || which == PH_R ||
                         which == PH_RC0;
  if (walks_psi) {
    for (int i = threadIdx.x; i < A.nst * kTile * kTile; i += blockDim.x) dyn_smem[i] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < A.nst; ++i) mb_init(&ring_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int NC = A.NC;
  switch (which) {
    case PH_INIT: {  // x = 0, r = b, NN2 inputs of b, b.b; NN2 up to d
      double acc = 0.0;
      for (long long q = gtid; q < A.NG; q += gstride) {
        const double bv = A.b[q];
        A.x[q] = 0.0;
        A.r[q] = bv;
        if (owned(A, q)) acc += bv * bv;
        write_local(A, q, bv);
      }
      const double bb = grid_sum(acc, A.part, 0, g, sm);
      if (leader) {
        A.xch[NC] = bb;
        A.st[ST_IT] = 0, A.st[ST_HL] = 0, A.st[ST_EXIT] = EX_RUN, A.st[ST_FIRST] = 1, A.st[ST_PFIRST] = 1;
      }
      ph_nn2a(A, R, sm, g, xs, xacc);
      break;
    }
    case PH_C0:
    case PH_RC0: {  // (start: ||b|| from the sums) then the rest of NN2
      if (which == PH_C0) {
        const double bnorm = sqrt(__ldcg(A.xch + NC));
        g.sync();
        if (leader) {
          A.sc[SC_BNORM] = bnorm;
          A.hist[0] = bnorm == 0.0 ? 0.0 : 1.0;
          A.st[ST_HL] = 1;
          if (bnorm == 0.0) A.st[ST_EXIT] = EX_ZERO;
        }
        if (bnorm == 0.0) break;
      }
      const double rz = ph_nn2b(A, R, sm, g, xs, xacc);
      if (leader) A.xch[NC + 2] = rz;
      break;
    }
    case PH_A: {  // complete z, beta, q_partial = S p_new, p.q partial
      for (long long t = gtid; t < (long long)A.H.n_shared * A.NT; t += gstride) {
        const int c = int(t % A.H.n_shared), j = int(t / A.H.n_shared);
        const long long q = (long long)j * A.n_iface + A.H.cnode[c];
        const double zq = halo_combine_one(A.H, c, j, A.z[q]);
        A.z[q] = zq;
        write_local_s(A, A.li_z, q, zq);
      }
      const double rz_new = __ldcg(A.xch + NC + 2);
      const bool first = A.st[ST_FIRST] != 0;
      const double beta = first ? 0.0 : rz_new / A.sc[SC_RZ];
      g.sync();
      if (leader) A.sc[SC_RZ] = rz_new, A.sc[SC_BETA] = beta, A.st[ST_PFIRST] = first, A.st[ST_FIRST] = 0;
      s_tiles_phase(A, R, sm, xs, xacc, 0, first, beta);
      g.sync();
      double acc = 0.0;
      for (long long q = gtid; q < A.NG; q += gstride) {
        const double y = s_reduce(A, q);
        A.q[q] = y;
        halo_pack_one(A.H, int(q / A.n_iface), int(q % A.n_iface), y);
        acc += y * (first ? A.z[q] : A.z[q] + beta * A.p[q]);
      }
      const double pq = grid_sum(acc, A.part, 1, g, sm);
      if (leader) A.xch[NC + 1] = pq;
      break;
    }
    case PH_B: {  // complete q; p, x, r updates; r.r; NN2 up to d
      for (long long t = gtid; t < (long long)A.H.n_shared * A.NT; t += gstride) {
        const int c = int(t % A.H.n_shared), j = int(t / A.H.n_shared);
        const long long q = (long long)j * A.n_iface + A.H.cnode[c];
        A.q[q] = halo_combine_one(A.H, c, j, A.q[q]);
      }
      const bool first = A.st[ST_PFIRST] != 0;
      const double beta = A.sc[SC_BETA], alpha = A.sc[SC_RZ] / __ldcg(A.xch + NC + 1);
      g.sync();
      double acc = 0.0;
      for (long long q = gtid; q < A.NG; q += gstride) {
        const double pn = first ? A.z[q] : A.z[q] + beta * A.p[q];
        A.p[q] = pn;
        write_local_s(A, A.li_p, q, pn);
        A.x[q] += alpha * pn;
        const double rn = A.r[q] - alpha * __ldcg(A.q + q);
        A.r[q] = rn;
        if (owned(A, q)) acc += rn * rn;
        write_local(A, q, rn);
      }
      const double rr = grid_sum(acc, A.part, 2, g, sm);
      if (leader) A.xch[NC] = rr;
      break;
    }
    case PH_B2: {  // convergence test (the loop condition; r.r summed over ranks), then NN2 up to d
      const int it = A.st[ST_IT] + 1, hl = A.st[ST_HL];
      const double rel = sqrt(__ldcg(A.xch + NC)) / A.sc[SC_BNORM];
      const int ex = rel <= A.tol ? EX_CHECK : (it >= A.max_iter ? EX_MAXIT : EX_RUN);
      g.sync();
      if (leader) {
        A.st[ST_IT] = it;
        if (ex != EX_CHECK) {  // a confirmed step records the true residual instead (verdict kernel)
          if (hl < A.hist_cap) A.hist[hl] = rel;
          A.st[ST_HL] = hl + 1;
        }
        A.st[ST_EXIT] = ex;
        if (ex != EX_RUN && A.use_cond) cudaGraphSetConditional(A.cond, 0);
      }
      if (ex != EX_RUN) break;  // converged / max_iter: no NN2 for this residual (src/pcg.cpp:30-44)
      ph_nn2a(A, R, sm, g, xs, xacc);
      break;
    }
    case PH_C: {  // the rest of NN2 (skipped once the test in PH_B2 ended the loop)
      if (A.st[ST_EXIT] != EX_RUN) break;
      const double rz = ph_nn2b(A, R, sm, g, xs, xacc);
      if (leader) A.xch[NC + 2] = rz;
      break;
    }
    case PH_T1: {  // q_partial = S x (true residual, src/pcg.cpp:31-40)
      for (long long q = gtid; q < A.NG; q += gstride) write_local_s(A, A.li_x, q, A.x[q]);
      g.sync();
      s_tiles_phase(A, R, sm, xs, xacc, 1, false, 0.0);
      g.sync();
      for (long long q = gtid; q < A.NG; q += gstride) {
        const double y = s_reduce(A, q);
        A.q[q] = y;
        halo_pack_one(A.H, int(q / A.n_iface), int(q % A.n_iface), y);
      }
      break;
    }
    case PH_T2: {  // r_true = b - S x (kept in q), its squared norm
      for (long long t = gtid; t < (long long)A.H.n_shared * A.NT; t += gstride) {
        const int c = int(t % A.H.n_shared), j = int(t / A.H.n_shared);
        const long long q = (long long)j * A.n_iface + A.H.cnode[c];
        A.q[q] = halo_combine_one(A.H, c, j, A.q[q]);
      }
      g.sync();
      double acc = 0.0;
      for (long long q = gtid; q < A.NG; q += gstride) {
        const double v = A.b[q] - __ldcg(A.q + q);
        A.q[q] = v;
        if (owned(A, q)) acc += v * v;
      }
      const double rt = grid_sum(acc, A.part, 3, g, sm);
      if (leader) A.xch[NC + 3] = rt;
      break;
    }
    case PH_R: {  // restart from the true residual (p kept): r = r_true, NN2 up to d
      for (long long q = gtid; q < A.NG; q += gstride) {
        const double v = __ldcg(A.q + q);
        A.r[q] = v;
        write_local(A, q, v);
      }
      if (leader) A.st[ST_EXIT] = EX_RUN;
      g.sync();
      ph_nn2a(A, R, sm, g, xs, xacc);
      break;
    }
    default:
      break;
  }
  if (threadIdx.x == 0)
    for (int c = R.consumed; c < R.issued; ++c) mb_wait(&R.full[c % R.nst], (c / R.nst) & 1);
  // the next walk's first tiles into L2 (a kernel boundary empties the ring;
  // the persistent kernel issues them across its grid barriers instead)
  if (A.ph_prefetch) {
    if (which == PH_A) l2_prefetch_range(A.rq, A.nst);                 // PH_B2: Q walk
    if (which == PH_B2 && NC > 0) l2_prefetch_range(A.rp, A.nst);      // PH_C: Psi walk
    if (which == PH_C || which == PH_RC0 || which == PH_C0) l2_prefetch_range(A.rs, A.nst);  // PH_A: S walk
  }
  __syncthreads();
}

// the true-residual verdict (src/pcg.cpp:31-40): converged, or restart
__global__ void pcg_phase_verdict_kernel(FusedPcg A) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double rel = sqrt(A.xch[A.NC + 3]) / A.sc[SC_BNORM];
  const int hl = A.st[ST_HL];
  if (hl < A.hist_cap) A.hist[hl] = rel;
  A.st[ST_HL] = hl + 1;
  A.st[ST_EXIT] = rel <= A.tol ? EX_CONV : EX_RESTART;
}

// --------------------------------------------------------------- host ----
// Contiguous tile ranges per CTA over a pack whose matrix s holds tiles
// [tile_base[s], tile_base[s + 1]) in row-major order: lower tiles of an
// nI x nI symmetric matrix (nJ empty), or all nI x nJ tiles (rectangular).
void RangeBufs::plan(const std::vector<long long>& tile_base, const std::vector<int>& nI, const std::vector<int>& nJ,
                     int grid) {
  const int nmat = int(nI.size());
  const bool rect = !nJ.empty();
  const long long n_tiles = tile_base[nmat];
  std::vector<long long> tf(grid + 1), pb(nmat + 1, 0);
  std::vector<int4> st(grid, make_int4(0, 0, 0, 0));
  std::vector<int> c0(nmat, 0), nc(nmat, 0);
  for (int c = 0; c <= grid; ++c) tf[c] = n_tiles * c / grid;
  auto cta_of = [&](long long t) {  // CTA whose (non-empty) range holds tile t
    return int(std::upper_bound(tf.begin(), tf.end(), t) - tf.begin()) - 1;
  };
  for (int c = 0; c < grid; ++c) {  // matrix, I, J of every CTA's first tile
    if (tf[c] >= tf[c + 1]) continue;
    const int s = int(std::upper_bound(tile_base.begin(), tile_base.end(), tf[c]) - tile_base.begin()) - 1;
    long long r = tf[c] - tile_base[s];
    int I = 0;
    if (rect) {
      I = int(r / nJ[s]), r %= nJ[s];
    } else {
      while (r > I) r -= ++I;  // row I holds I + 1 tiles
    }
    st[c] = make_int4(s, I, int(r), 0);
  }
  for (int s = 0; s < nmat; ++s) {  // CTAs covering each matrix and its partials
    if (tile_base[s + 1] > tile_base[s]) {
      const int a = cta_of(tile_base[s]), b = cta_of(tile_base[s + 1] - 1);
      c0[s] = a, nc[s] = b - a + 1;
    }
    pb[s + 1] = pb[s] + (long long)nc[s] * kTile * (nI[s] + (rect ? nJ[s] : 0));
  }
  t_first.upload(tf), start.upload(st);
  this->c0.upload(c0), ncta.upload(nc), pbase.upload(pb);
  h_pbase = pb, h_ncta = nc;
  part.alloc(std::max<long long>(1, pb[nmat]));
  SGW_CUDA(cudaMemset(part.p, 0, part.n * sizeof(double)));  // slots of CTAs with empty ranges stay 0
}

// Psi_s (column-major r_s x c_s) -> tile (I, J) = column-major 64 x w chunk of
// columns [64 I, 64 I + w), rows [64 J, 64 J + 64) (zeros past r_s).  One CTA per tile.
__global__ void psi_tiles_kernel(const double* __restrict__ Psi, const long long* __restrict__ psioff,
                                 const int4* __restrict__ desc, const long long* __restrict__ toff,
                                 const int* __restrict__ nr, const int* __restrict__ nc, int nt,
                                 double* __restrict__ tiles) {
  const int4 d = desc[blockIdx.x];  // {s, I, J, w}
  const int rs = nt * nr[d.x];
  const double* src = Psi + psioff[d.x];
  double* dst = tiles + toff[blockIdx.x];
  for (int e = threadIdx.x; e < d.w * kTile; e += blockDim.x) {
    const int c = 64 * d.y + e / kTile, r = 64 * d.z + e % kTile;
    dst[e] = r < rs ? src[(long long)c * rs + r] : 0.0;
  }
}

void GpuSolver::build_psi_tiles() {
  std::vector<int> nI(NS), nJ(NS);
  std::vector<long long> base(NS + 1, 0), toff;
  std::vector<int> bytes;
  std::vector<int4> desc;
  long long off = 0;
  for (int s = 0; s < NS; ++s) {
    const int cs = NT * nc_[s];
    nI[s] = cdiv(cs, kTile), nJ[s] = Qp.ntile[s];  // Qp: the r_s = NT nr_s remaining dofs
    for (int I = 0; I < nI[s]; ++I)
      for (int J = 0; J < nJ[s]; ++J) {
        const int w = std::min(kTile, cs - kTile * I);
        desc.push_back(make_int4(s, I, J, w));
        toff.push_back(off);
        bytes.push_back(w * kTile * 8);
        off += (long long)w * kTile;
      }
    base[s + 1] = (long long)desc.size();
  }
  psi_nI_ = nI, psi_nJ_ = nJ;
  psi_tiles_.alloc(std::max<long long>(1, off));
  psi_toff_.upload(toff), psi_tbytes_.upload(bytes), psi_dnI_.upload(nI), psi_dnJ_.upload(nJ);
  if (!desc.empty()) {
    DBuf<int4> d;
    d.upload(desc);
    psi_tiles_kernel<<<(unsigned)desc.size(), 256, 0, st_>>>(Psi.p, d_psioff.p, d.p, psi_toff_.p, nr_d.p, nc_d.p, NT,
                                                             psi_tiles_.p);
    SGW_LAUNCHED();
    SGW_CUDA(cudaStreamSynchronize(st_));
  }
  rp_.plan(base, nI, nJ, fused_grid_);
}

void GpuSolver::setup_fused_pcg() {
  tphase_.alloc(8), tphase_.zero(st_);
  if (P.implicit_schur || direct_) {  // reduced-memory: the host-driven loop without S tiles; direct: no PCG
    use_fused_ = false;
    if (direct_) use_phase_ = walk_ok_ = false;
    return;
  }
  int dev = 0, sms = 0, nb = 0, smem_sm = 0, smem_blk = 0;
  SGW_CUDA(cudaGetDevice(&dev));
  SGW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SGW_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  SGW_CUDA(cudaDeviceGetAttribute(&smem_blk, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // shared memory per CTA: the tile ring, the local input vector and the
  // accumulator of the longest local vector (S_s, Q_s, or [corners | remaining
  // dofs] of Psi_s).  Default two CTAs per SM (more warps for the scatter
  // phases; measured 0.56 vs 0.64 ms per C2 iteration with one CTA and a
  // deeper ring) if each gets >= 2 stages, else one with the deepest ring
  // that fits.  SGW_PCG_BPS / SGW_PCG_RING tune.
  fused_maxlen_ = 0;
  for (int s = 0; s < NS; ++s)
    fused_maxlen_ = std::max({fused_maxlen_, kTile * Sp.ntile[s], kTile * (Qp.ntile[s] + cdiv(NT * nc_[s], kTile))});
  cudaFuncAttributes fa{};
  SGW_CUDA(cudaFuncGetAttributes(&fa, (const void*)pcg_fused_kernel));
  // small tile sets (C1: 12 MB per iteration) are latency-bound: one CTA per
  // SM halves the CTA partials every scatter sums and the grid-barrier cost
  // (measured at C1: 61 vs 73 us per iteration; at C2 two CTAs per SM win,
  // 0.54 vs 0.64 ms)
  int bps = bytes_S() + bytes_Q() < 64e6 ? 1 : 2;
  if (const char* e = std::getenv("SGW_PCG_BPS")) bps = std::max(1, std::atoi(e));
  const long long vec = 2LL * fused_maxlen_ * 8;
  for (;; --bps) {
    const long long avail = std::min<long long>(smem_blk, smem_sm / bps - 1024) - (long long)fa.sharedSizeBytes - vec;
    fused_nst_ = (int)std::min<long long>(kMaxRing, avail / kTileBytes);
    if (fused_nst_ >= 2 || bps == 1) break;
  }
  if (const char* e = std::getenv("SGW_PCG_RING")) fused_nst_ = std::min(kMaxRing, std::atoi(e));
  if (fused_nst_ < 1) {
    // a subdomain's local interface vectors exceed one CTA's shared memory
    // (very large PCE bases, e.g. P+1 = 153 on 32 x 32 subdomains): the
    // host-driven PCG with the per-tile S / Q products, which keep no whole
    // local vector in shared memory
    use_fused_ = use_phase_ = walk_ok_ = false;
    return;
  }
  fused_smem_ = (size_t)fused_nst_ * kTileBytes + (size_t)vec;
  ensure_dyn_smem((const void*)pcg_fused_kernel, fused_smem_);
  SGW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pcg_fused_kernel, 256, fused_smem_));
  {  // the phase-split kernel walks the same CTA ranges: same grid, co-resident too
    int nb2 = 0;
    ensure_dyn_smem((const void*)pcg_phase_kernel, fused_smem_);
    SGW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb2, pcg_phase_kernel, 256, fused_smem_));
    nb = std::min(nb, nb2);
  }
  fused_grid_ = std::max(1, std::min(nb, bps)) * sms;
  if (const char* e = std::getenv("SGW_PCG_GRID"))  // tuning hook (<= the co-resident maximum)
    fused_grid_ = std::max(1, std::min(fused_grid_, std::atoi(e)));
  ensure_dyn_smem((const void*)walk_kernel, fused_smem_);
  rs_.plan(Sp.tile_base, Sp.ntile, {}, fused_grid_);
  rq_.plan(Qp.tile_base, Qp.ntile, {}, fused_grid_);
  walk_ok_ = true;  // the host-driven loop streams S / Q / Psi with walk_kernel too
  build_psi_tiles();
  build_scatter_desc();
  {  // tiles of S, Q and Psi within ~half of L2 (C1: 12 MB): keep them resident
    const double tile_bytes = bytes_S() + bytes_Q();
    l2_keep_ = tile_bytes <= 48e6 ? 1 : 0;
    if (const char* e = std::getenv("SGW_PCG_L2KEEP")) l2_keep_ = std::atoi(e) != 0;  // tuning hook
  }
  {
    std::vector<int> ncs(NS);
    for (int s = 0; s < NS; ++s) ncs[s] = NT * nc_[s];
    psi_ncs_.upload(ncs);
  }
  ucl_.alloc(std::max<long long>(1, coff_.back())), ucl_.zero(st_);
  fused_part_.alloc(size_t(8) * fused_grid_);
  fused_out_.alloc(4);
  fused_hist_.alloc(P.max_iter + 8);
  for (DBuf<double>* b : {&li_z_, &li_p_, &li_xx_}) b->alloc(Sp.xlen), b->zero(st_);  // padding stays 0
  ph_xch_.alloc(NC + 8), ph_xch_.zero(st_);
  ph_sc_.alloc(8), ph_sc_.zero(st_);
  ph_st_.alloc(8), ph_st_.zero(st_);
  // sharded runs (and SGW_PCG=phase): the phase-split PCG; SGW_PCG=host: the host-driven loop
  const char* e = std::getenv("SGW_PCG");
  const std::string mode = e ? e : "";
  use_fused_ = !comm_ && mode != "host" && mode != "phase";
  use_phase_ = mode != "host";
}

void GpuSolver::build_scatter_desc() {
  const int ni = G.n_iface;
  std::vector<int4> ifd(4 * (size_t)ni, make_int4(-1, 0, 0, 0)), sred(4 * (size_t)ni, make_int4(0, 0, 0, 0));
  std::vector<int4> zred(4 * (size_t)ni, make_int4(0, 0, 0, -2)), pred(4 * (size_t)ni, make_int4(0, 0, 0, 0));
  std::vector<double> ifw(4 * (size_t)ni, 0.0);
  std::vector<int> cnt(ni, 0);
  auto i32 = [](long long v) {
    if (v < 0 || v >= (1LL << 31)) throw Error(1, "PCG glue descriptor out of 32-bit range");
    return int(v);
  };
  for (int s = 0; s < NS; ++s) {  // ascending s: the reference's reduction order
    const auto& sd = G.sub[s];
    std::vector<int> kind(ng_[s], 0);
    for (int r = 0; r < nr_[s]; ++r) kind[sd.r_local[r]] = r;
    for (int c = 0; c < nc_[s]; ++c) kind[sd.c_local[c]] = -1 - c;
    for (int pp = 0; pp < ng_[s]; ++pp) {
      const int gq = sd.iface_pos[pp], e = cnt[gq]++;
      if (e >= 4) throw Error(1, "more than four subdomains share an interface node");
      const size_t k = 4 * (size_t)gq + e;
      const int kd = kind[pp];
      ifd[k] = make_int4(i32(Sp.xoff[s] + pp), ng_[s], i32(kd >= 0 ? roff_[s] + kd : coff_[s] + (-1 - kd)),
                         kd >= 0 ? nr_[s] : -nc_[s]);
      ifw[k] = sd.w[pp];
      sred[k] = make_int4(i32(rs_.h_pbase[s] + pp), ng_[s], kTile * Sp.ntile[s], rs_.h_ncta[s]);
      if (kd >= 0) {
        zred[k] = make_int4(i32(rq_.h_pbase[s] + kd), nr_[s], kTile * Qp.ntile[s], rq_.h_ncta[s]);
        if (!psi_nI_.empty() && !rp_.h_pbase.empty())
          pred[k] = make_int4(i32(rp_.h_pbase[s] + (long long)kTile * psi_nI_[s] + kd), nr_[s],
                              kTile * (psi_nI_[s] + psi_nJ_[s]), rp_.h_ncta[s]);
      } else {
        zred[k] = make_int4(i32(coff_[s] + (-1 - kd)), nc_[s], 0, -1);
      }
    }
  }
  d_ifd_.upload(ifd), d_ifw_.upload(ifw), d_sred_.upload(sred), d_zred_.upload(zred), d_pred_.upload(pred);
}

FusedPcg GpuSolver::fused_args(const double* b, double* x) const {
  FusedPcg A{};
  A.NG = NG;
  A.n_iface = G.n_iface, A.NT = NT, A.NS = NS, A.n_corner = G.n_corner, A.NC = NC;
  A.max_iter = P.max_iter, A.hist_cap = (int)fused_hist_.n, A.tol = P.tol;
  A.b = b, A.x = x, A.r = vr.p, A.z = vz.p, A.p = vp.p, A.q = vq.p;
  A.s_xoff = Sp.d_xoff.p, A.q_xoff = Qp.d_xoff.p;
  A.fr = r_x.p, A.fc = c_f.p;
  A.inv_cnt = inv_cnt.p, A.inv_s = inv_s.p, A.inv_p = inv_p.p, A.ip_off = ip_off.p, A.ng = ng_d.p, A.nr = nr_d.p,
  A.nc = nc_d.p, A.pkind = pkind_.p, A.iface_w = iface_w.p;
  A.cinv_cnt = cinv_cnt.p, A.cinv_s = cinv_s.p, A.cinv_c = cinv_c.p;
  A.roff = d_roff.p, A.coff = d_coff.p;
  A.Finv = Finv.p, A.dco = dcoarse.p, A.uco = ucoarse.p, A.ucl = ucl_.p;
  A.part = fused_part_.p, A.out = fused_out_.p, A.hist = fused_hist_.p;
  A.li_z = li_z_.p, A.li_p = li_p_.p, A.li_x = li_xx_.p;
  A.tphase = KP.on ? tphase_.p : nullptr;
  A.rs = RangePack{Sp.tiles.p, nullptr, nullptr, Sp.d_ntile.p, nullptr, 0, rs_.t_first.p, rs_.start.p, rs_.c0.p,
                   rs_.ncta.p, rs_.pbase.p, rs_.part.p};
  A.rq = RangePack{Qp.tiles.p, nullptr, nullptr, Qp.d_ntile.p, nullptr, 0, rq_.t_first.p, rq_.start.p, rq_.c0.p,
                   rq_.ncta.p, rq_.pbase.p, rq_.part.p};
  A.rp = RangePack{psi_tiles_.p, psi_toff_.p, psi_tbytes_.p, psi_dnI_.p, psi_dnJ_.p, 1, rp_.t_first.p, rp_.start.p,
                   rp_.c0.p, rp_.ncta.p, rp_.pbase.p, rp_.part.p};
  A.nst = fused_nst_, A.maxlen = fused_maxlen_;
  A.H = halo_dev();
  A.own = dot_mask();
  A.xch = ph_xch_.p, A.sc = ph_sc_.p, A.st = ph_st_.p;
  A.cond = 0, A.use_cond = 0;
  A.l2_keep = l2_keep_;
  A.ph_prefetch = 0;  // measured: 0.565 vs 0.560 ms per C2 iteration with it (the prefetches compete)
  if (const char* e = std::getenv("SGW_PHASE_PREFETCH")) A.ph_prefetch = std::atoi(e);  // tuning hook
  A.ifd = d_ifd_.p, A.ifw = d_ifw_.p, A.sred = d_sred_.p, A.zred = d_zred_.p, A.pred = d_pred_.p;
  return A;
}

// ------------------------------------------------ phase-split PCG (host) --
// Sequences of the phase-split solve (see pcg_phase_kernel).  xch layout:
// [0, NC) d, NC r.r | b.b, NC+1 p.q, NC+2 r.z, NC+3 rt.rt.
void GpuSolver::phase_seq(int which, const FusedPcg& A0) {
  FusedPcg A = A0;
  static const bool timing = std::getenv("SGW_PHASE_TIMING") != nullptr;  // diagnostics: per-phase event timing
  static cudaEvent_t te[2];
  static double tsum[16];
  static int tcnt[16];
  if (timing && !te[0]) cudaEventCreate(&te[0]), cudaEventCreate(&te[1]);
  auto K = [&](int ph) {
    void* args[] = {&A, &ph};
    if (timing) cudaEventRecord(te[0], st_);
    SGW_CUDA(cudaLaunchCooperativeKernel((const void*)pcg_phase_kernel, dim3(fused_grid_), dim3(256), args,
                                         fused_smem_, st_));
    SGW_LAUNCHED();
    if (timing) {
      cudaEventRecord(te[1], st_);
      cudaEventSynchronize(te[1]);
      float ms = 0;
      cudaEventElapsedTime(&ms, te[0], te[1]);
      tsum[ph] += ms, ++tcnt[ph];
      if (tcnt[PH_A] % 40 == 0 && ph == PH_C)
        for (int k = 0; k < 10; ++k)
          if (tcnt[k]) std::fprintf(stderr, "phase %d: %d launches, %.1f us avg\n", k, tcnt[k], 1e3 * tsum[k] / tcnt[k]);
    }
  };
  auto AR = [&](int off, int cnt) {
    if (comm_) comm_->allreduce_sum(ph_xch_.p + off, cnt, st_);
  };
  auto XH = [&]() {
    if (comm_ && !G.halo.peers.empty()) halo_exchange();
  };
  switch (which) {
    case 0:  // start: x = 0, r = b, z = NN2(b), r.z
      K(PH_INIT), AR(0, NC + 1), K(PH_C0), XH(), AR(NC + 2, 1);
      break;
    case 1:  // one iteration
      K(PH_A), XH(), AR(NC + 1, 1), K(PH_B), AR(NC, 1), K(PH_B2), AR(0, NC), K(PH_C), XH(), AR(NC + 2, 1);
      break;
    case 2:  // true residual and its verdict
      K(PH_T1), XH(), K(PH_T2), AR(NC + 3, 1);
      pcg_phase_verdict_kernel<<<1, 32, 0, st_>>>(A);
      SGW_LAUNCHED();
      break;
    case 3:  // restart from the true residual
      K(PH_R), AR(0, NC), K(PH_RC0), XH(), AR(NC + 2, 1);
      break;
  }
}

// Graphs of the four sequences; the iteration is the body of a WHILE
// conditional node (the loop condition is set by the PH_C kernel), so a solve
// runs without host synchronisation until the recurrence residual meets the
// tolerance.  Rebuilt when the solve's b / x buffers change.
bool GpuSolver::build_phase_graphs(const double* b, double* x) {
  for (auto& ge : ph_graph_)
    if (ge) cudaGraphExecDestroy(ge), ge = nullptr;
  ph_graph_b_ = b, ph_graph_x_ = x;
  const bool kp = KP.on;
  KP.on = false;
  const FusedPcg A = fused_args(b, x);
  bool ok = true;
  const long long l0 = g_launches.load();
  for (int k = 0; k < 4 && ok; ++k) {
    const long long c0 = g_launches.load();
    cudaGraph_t gr = nullptr;
    if (k == 1) {  // WHILE { iteration }
      ok = cudaGraphCreate(&gr, 0) == cudaSuccess;
      cudaGraphConditionalHandle h = 0;
      ok = ok && cudaGraphConditionalHandleCreate(&h, gr, 1, cudaGraphCondAssignDefault) == cudaSuccess;
      cudaGraphNodeParams cp{};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t node;
      ok = ok && cudaGraphAddNode(&node, gr, nullptr, 0, &cp) == cudaSuccess;
      if (ok) {
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        FusedPcg Ab = A;
        Ab.cond = h, Ab.use_cond = 1;
        ok = cudaStreamBeginCaptureToGraph(st_, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) ==
             cudaSuccess;
        if (ok) {
          try {
            phase_seq(1, Ab);
          } catch (const Error&) {
            ok = false;
          }
          cudaGraph_t out = nullptr;
          ok = cudaStreamEndCapture(st_, &out) == cudaSuccess && ok;
        }
      }
    } else {
      ok = cudaStreamBeginCapture(st_, cudaStreamCaptureModeRelaxed) == cudaSuccess;
      if (ok) {
        try {
          phase_seq(k, A);
        } catch (const Error&) {
          ok = false;
        }
        ok = cudaStreamEndCapture(st_, &gr) == cudaSuccess && ok;
      }
    }
    ok = ok && cudaGraphInstantiate(&ph_graph_[k], gr, 0) == cudaSuccess;
    if (gr) cudaGraphDestroy(gr);
    ph_graph_launches_[k] = g_launches.load() - c0;
  }
  g_launches = l0;  // counted per replay
  KP.on = kp;
  if (!ok) {
    cudaGetLastError();  // clear a capture / instantiation failure: fall back to stream launches
    for (auto& ge : ph_graph_)
      if (ge) cudaGraphExecDestroy(ge), ge = nullptr;
    ph_graph_b_ = nullptr, ph_graph_x_ = nullptr;
  }
  return ok;
}

int GpuSolver::pcg_phase(const double* b, double* x, bool* converged, std::vector<double>* hist) {
  cudaEventRecord(ev_[0], st_);
  if (!h_st_) SGW_CUDA(cudaMallocHost(&h_st_, 8 * sizeof(int)));
  const bool graphs = (!comm_ || comm_->capturable()) && ph_graph_ok_ && !std::getenv("SGW_PHASE_NOGRAPH");
  if (graphs && (ph_graph_b_ != b || ph_graph_x_ != x || !ph_graph_[0]))
    ph_graph_ok_ = build_phase_graphs(b, x);
  const bool use_graphs = graphs && ph_graph_ok_;
  const FusedPcg A = fused_args(b, x);
  auto run = [&](int k) {
    if (use_graphs) {
      SGW_CUDA(cudaGraphLaunch(ph_graph_[k], st_));
      g_launches += ph_graph_launches_[k];
    } else {
      phase_seq(k, A);
    }
  };
  auto state = [&]() {
    SGW_CUDA(cudaMemcpyAsync(h_st_, ph_st_.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, st_));
    SGW_CUDA(cudaStreamSynchronize(st_));
    if (comm_) comm_->poll();
    return h_st_[ST_EXIT];
  };
  auto loop = [&]() {
    if (use_graphs) {
      run(1);
      return state();
    }
    for (;;) {  // host-driven iterations (non-capturable exchange): one state read per iteration
      run(1);
      const int ex = state();
      if (ex != EX_RUN) return ex;
    }
  };
  run(0);
  int ex = state();
  bool conv = false;
  if (ex == EX_ZERO) {
    conv = true;
  } else {
    for (;;) {
      ex = loop();
      if (ex != EX_CHECK) break;  // max_iter without meeting the tolerance
      run(2);
      ex = state();
      if (ex == EX_CONV) {
        conv = true;
        break;
      }
      if (h_st_[ST_IT] >= P.max_iter) break;
      run(3);
    }
  }
  cudaEventRecord(ev_[1], st_);
  SGW_CUDA(cudaEventSynchronize(ev_[1]));
  float ms = 0;
  cudaEventElapsedTime(&ms, ev_[0], ev_[1]);
  const int it = h_st_[ST_IT], hl = std::min<int>(h_st_[ST_HL], (int)fused_hist_.n);
  T.pcg_ms += ms;
  T.iterations += it;
  T.matvecs += it;
  T.nn2s += it;
  std::vector<double> h(hl);
  if (hl) SGW_CUDA(cudaMemcpy(h.data(), fused_hist_.p, hl * sizeof(double), cudaMemcpyDeviceToHost));
  last_rel = hl ? h.back() : 0.0;
  if (hist) *hist = std::move(h);
  *converged = conv;
  return it;
}

RangePack GpuSolver::range_pack(int which) const {
  const TilePack& tp = which == 0 ? Sp : Qp;
  const RangeBufs& rb = which == 0 ? rs_ : rq_;
  return RangePack{tp.tiles.p, nullptr, nullptr, tp.d_ntile.p, nullptr, 0, rb.t_first.p, rb.start.p, rb.c0.p,
                   rb.ncta.p, rb.pbase.p, rb.part.p};
}

// the Psi^T tile walk for the host-driven NN2: pass 1 on [0 | f_r], pass 2 on [B_s u_c | 0]
void GpuSolver::walk_psi(int pass, const double* x) {
  if (!rp_.t_first.p) return;
  const RangePack P{psi_tiles_.p, psi_toff_.p, psi_tbytes_.p, psi_dnI_.p, psi_dnJ_.p, 1, rp_.t_first.p, rp_.start.p,
                    rp_.c0.p, rp_.ncta.p, rp_.pbase.p, rp_.part.p};
  walk_kernel<<<fused_grid_, 256, fused_smem_, st_>>>(P, x, pass == 1 ? d_roff.p : d_coff.p, fused_nst_, fused_maxlen_,
                                                      pass, psi_ncs_.p);
  SGW_LAUNCHED();
}

RangePack GpuSolver::psi_pack() const {
  return RangePack{psi_tiles_.p, psi_toff_.p, psi_tbytes_.p, psi_dnI_.p, psi_dnJ_.p, 1, rp_.t_first.p, rp_.start.p,
                   rp_.c0.p, rp_.ncta.p, rp_.pbase.p, rp_.part.p};
}

void GpuSolver::walk_pack(int which, const double* x) {
  const TilePack& tp = which == 0 ? Sp : Qp;
  if (!tp.n_tiles) return;
  cudaEvent_t e0;
  KP.begin(which == 0 ? K_SYMV_S : K_SYMV_Q, st_, &e0);
  walk_kernel<<<fused_grid_, 256, fused_smem_, st_>>>(range_pack(which), x, tp.d_xoff.p, fused_nst_, fused_maxlen_, 0,
                                                      nullptr);
  SGW_LAUNCHED();
  KP.end(st_);
}

int GpuSolver::pcg_fused(const double* b, double* x, bool* converged, std::vector<double>* hist) {
  pcg_fused_launch(b, x);
  SGW_CUDA(cudaEventSynchronize(ev_[6]));
  return pcg_fused_finish(converged, hist);
}

// Asynchronous half: the kernel, then its outputs (iterations, convergence,
// residual history) copied into pinned host memory; pcg_fused_finish reads them
// once the stream has passed ev_[6] (step() launches the recovery first).
void GpuSolver::pcg_fused_launch(const double* b, double* x) {
  if (!h_fused_) SGW_CUDA(cudaMallocHost(&h_fused_, (4 + fused_hist_.n) * sizeof(double)));
  cudaEventRecord(ev_[0], st_);
  FusedPcg A = fused_args(b, x);
  void* args[] = {&A};
  SGW_CUDA(cudaLaunchCooperativeKernel((const void*)pcg_fused_kernel, dim3(fused_grid_), dim3(256), args,
                                       fused_smem_, st_));
  SGW_LAUNCHED();
  cudaEventRecord(ev_[1], st_);  // end of the solve (the PCG time)
  // the read-back runs on a side stream: the step's recovery kernels follow the
  // solve on st_ without waiting for two small device-to-host copies
  if (!side_) SGW_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
  SGW_CUDA(cudaStreamWaitEvent(side_, ev_[1], 0));
  SGW_CUDA(cudaMemcpyAsync(h_fused_, fused_out_.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, side_));
  SGW_CUDA(cudaMemcpyAsync(h_fused_ + 4, fused_hist_.p, fused_hist_.n * sizeof(double), cudaMemcpyDeviceToHost, side_));
  cudaEventRecord(ev_[6], side_);  // outputs in pinned memory
}

int GpuSolver::pcg_fused_finish(bool* converged, std::vector<double>* hist) {
  int out[3];
  std::memcpy(out, h_fused_, sizeof(out));
  float ms = 0;
  cudaEventElapsedTime(&ms, ev_[0], ev_[1]);
  T.pcg_ms += ms;
  T.iterations += out[0];
  T.matvecs += out[0];
  T.nn2s += out[0];
  *converged = out[1] != 0;
  const int hl = std::min<int>(out[2], (int)fused_hist_.n);
  last_rel = hl > 0 ? h_fused_[4 + hl - 1] : 0.0;
  if (hist) hist->assign(h_fused_ + 4, h_fused_ + 4 + hl);
  return out[0];
}

}  // namespace sgw
