// Device pieces of the packed-symmetric 64x64-tile SYMV shared by the
// standalone kernels (pcg.cu) and the persistent PCG kernel (pcg_fused.cu).
#pragma once

#include "common.cuh"

namespace sgw {

// One 64x64 lower tile T_IJ (row-major, diagonal tiles stored full) times the
// 64-vectors xI / xJ (shared memory), by 256 threads (8 warps x 8 rows):
//   rowpart = T_IJ xJ ;  colpart = T_IJ^T xI (I != J).
// Warp w streams rows 8w..8w+7 with 128-bit loads (one 512-byte row per warp
// load); the 8 row sums use a butterfly multi-row reduction over the lanes.
// csum: __shared__ double[8][64] scratch.
__device__ __forceinline__ void tile_symv(const double* __restrict__ T, const double* xI, const double* xJ,
                                          bool diag, double* __restrict__ rowpart, double* __restrict__ colpart,
                                          double (*csum)[kTile]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double2* T2 = reinterpret_cast<const double2*>(T);
  double2 v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = __ldcs(T2 + (w * 8 + q) * (kTile / 2) + lane);
  const double2 xj = reinterpret_cast<const double2*>(xJ)[lane];
  const double* xi = xI + w * 8;
  double rs[8], c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    rs[q] = v[q].x * xj.x + v[q].y * xj.y;
    const double xv = xi[q];
    c0 += v[q].x * xv;
    c1 += v[q].y * xv;
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
    rowpart[w * 8 + row] = rs[0];
  }
  if (!diag) {
    csum[w][2 * lane] = c0;
    csum[w][2 * lane + 1] = c1;
    __syncthreads();
    if (threadIdx.x < kTile) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) s += csum[k][threadIdx.x];
      colpart[threadIdx.x] = s;
    }
  }
}

// y_s[i] of matrix s from the tile partials, fixed order: row partials of
// tiles (I, 0..I), then column partials of tiles (I+1..nt-1, I).
__device__ __forceinline__ double tile_reduce(const double* __restrict__ rowpart, const double* __restrict__ colpart,
                                              long long base, int nt, int i) {
  const int I = i / kTile, r = i % kTile;
  const double* rp = rowpart + (base + (long long)I * (I + 1) / 2) * kTile + r;
  // the partials were written by other CTAs before a grid barrier: L2 loads,
  // issued 8 at a time (the sum order stays J ascending, then K ascending)
  constexpr int U = 8;
  double s = 0.0;
  int J = 0;
  for (; J + U <= I + 1; J += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(rp + (long long)(J + u) * kTile);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
  }
  for (; J <= I; ++J) s += __ldcg(rp + (long long)J * kTile);
  const double* cp = colpart + (base + I) * kTile + r;  // tile (K, I) at base + K(K+1)/2 + I
  int K = I + 1;
  for (; K + U <= nt; K += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(cp + (long long)(K + u) * (K + u + 1) / 2 * kTile);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
  }
  for (; K < nt; ++K) s += __ldcg(cp + (long long)K * (K + 1) / 2 * kTile);
  return s;
}

// A tile pack walked in contiguous tile ranges, one per CTA.  Two kinds:
//  * symmetric (S_s, Q_s): lower 64x64 tiles (I, J <= I), row-major over the
//    tiles of a matrix, diagonal tiles full, 32 KB each;
//  * rectangular (Psi_s^T): tiles (I, J), I over 64-wide corner-column chunks,
//    J over 64-row blocks of the remaining dofs, row-major; tile (I, J) is the
//    column-major 64 x w chunk of Psi_s (w = the chunk's valid columns, rows
//    past r_s stored as zeros), i.e. row-major Psi^T rows of stride 64, w x 512
//    bytes, so one bulk copy moves only stored data.
// A CTA keeps the local input vector of its current matrix and a local
// accumulator in shared memory, adds every tile's row and column products
// into it (tile_acc), and at a matrix boundary writes the accumulator as its
// partial of that matrix: y_s = sum over the CTAs covering s of their
// partials, in CTA order.  Local vectors: symmetric [64 nt]; rectangular
// [64 nI (corner chunks) | 64 nJ (remaining-dof blocks)].
struct RangePack {
  const double* tiles;
  const long long* toff;      // per tile: offset in doubles (null: t * 4096)
  const int* tbytes;          // per tile: bytes (null: 32 KB)
  const int* nI;              // per matrix: tile rows (symmetric: tiles per side)
  const int* nJ;              // per matrix: tile columns (rectangular only)
  int rect;
  const long long* t_first;   // [G + 1] first tile of each CTA's range
  const int4* start;          // [G] {matrix, I, J} of each CTA's first tile
  const int* c0;              // per matrix: first CTA covering it
  const int* ncta;            // per matrix: CTAs covering it
  const long long* pbase;     // per matrix: offset of its partials in part
  double* part;               // partials [pbase[s] + (c - c0[s]) len_s + i]
};

// sum of the n CTA partials p[k len] of one local entry, k ascending
__device__ __forceinline__ double partial_sum(const double* p, int len, int n) {
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
// NL partial lists summed side by side: list e is what partial_sum(p[e], len[e],
// n[e]) returns (k ascending, the same additions in the same order), but the
// loads of all lists are in flight together, KU entries of each per round, instead of one
// list after the other.  An interface node's reduction is then a few L2 round
// trips, not (slots x lists x n / 4): that chain was most of the scatter phases
// of small problems (C1).  Empty lists (n <= 0) load nothing.
template <int NL, int KU>
__device__ __forceinline__ void partial_sums(const double* const (&p)[NL], const int (&len)[NL], const int (&n)[NL],
                                             double (&y)[NL]) {
  int nmax = 0;
#pragma unroll
  for (int e = 0; e < NL; ++e) y[e] = 0.0, nmax = max(nmax, n[e]);
  for (int k = 0; k < nmax; k += KU) {
    double a[KU][NL];
#pragma unroll
    for (int u = 0; u < KU; ++u)
#pragma unroll
      for (int e = 0; e < NL; ++e) a[u][e] = k + u < n[e] ? __ldcg(p[e] + (long long)(k + u) * len[e]) : 0.0;
#pragma unroll
    for (int u = 0; u < KU; ++u)
#pragma unroll
      for (int e = 0; e < NL; ++e)
        if (k + u < n[e]) y[e] += a[u][e];
  }
}
// y_s[i] from the partials of the CTAs covering symmetric matrix s
__device__ __forceinline__ double range_reduce(const RangePack& P, int s, int i) {
  return partial_sum(P.part + P.pbase[s] + i, kTile * P.nI[s], P.ncta[s]);
}
// Psi^T x (corner part, i < 64 nI) or Psi x (remaining-dof part, offset 64 nI)
// of rectangular matrix s
__device__ __forceinline__ double rect_reduce(const RangePack& P, int s, int i) {
  return partial_sum(P.part + P.pbase[s] + i, kTile * (P.nI[s] + P.nJ[s]), P.ncta[s]);
}

// Halo of the shared interface nodes (host.hpp Halo) on the device.  Send /
// receive buffers hold one block per peer, term-major inside a block
// ([j * cnt + i], cnt = the peer's shared nodes).
//  * pack: node q's partial of term j goes to send[e.x + j * e.y] for every
//    entry e of pk[pk_ptr[q] .. pk_ptr[q + 1]) (one per peer sharing q);
//  * combine: shared node cnode[c] = sum over its sources in ascending rank,
//    csrc[..] = {offset in recv (or -1: this rank's own partial), stride}.
// Every holder of a node sums the same values in the same order, so the
// completed vectors are bitwise identical on all ranks.
struct HaloDev {
  int nloc;              // local interface nodes (vector stride per term)
  int n_shared;          // shared nodes
  const int* pk_ptr;     // nloc + 1
  const int2* pk;        // {base + i, cnt}
  const int* cnode;      // n_shared
  const int* cptr;       // n_shared + 1
  const int2* csrc;      // {recv offset | -1, stride}
  double* send;
  const double* recv;
};

// partial y (term j, local node gq) into the send blocks of the peers sharing gq
__device__ __forceinline__ void halo_pack_one(const HaloDev& H, int j, int gq, double y) {
  for (int e = H.pk_ptr[gq]; e < H.pk_ptr[gq + 1]; ++e) {
    const int2 d = H.pk[e];
    H.send[d.x + (long long)j * d.y] = y;
  }
}
// completed value of shared node c (term j) from the own partial `own`
__device__ __forceinline__ double halo_combine_one(const HaloDev& H, int c, int j, double own) {
  double acc = 0.0;
  for (int e = H.cptr[c]; e < H.cptr[c + 1]; ++e) {
    const int2 d = H.csrc[e];
    acc += d.x < 0 ? own : __ldcg(H.recv + d.x + (long long)j * d.y);
  }
  return acc;
}

}  // namespace sgw
