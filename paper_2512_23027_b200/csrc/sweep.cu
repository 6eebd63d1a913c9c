// Batched interior Dirichlet solve x <- A_II^-1 x for every subdomain
// (src/sg.cpp:317 and :350: SimplicialLLT::solve, restated block-wise).
//
// A_II is block tridiagonal over the H interior grid rows (blocks B = W (P+1),
// node-major / term-minor).  The solve is the block Thomas algorithm on the
// Schur complements D_k = L_kk L_kk^T of the block Cholesky factor:
//   forward   w_0 = b_0,  z_k = D_k^-1 w_k,  w_{k+1} = b_{k+1} - A_{k+1,k} z_k
//   backward  x_{H-1} = z_{H-1},  x_k = D_k^-1 (w_k - A_{k,k+1} x_{k+1})
// D_k^-1 = L_kk^-T L_kk^-1 is symmetric and stored once (lower 64 x 64 tiles,
// row-major, swizzled by sw_col, diagonal tiles full); the grid-row coupling A_{k+1,k} only joins a
// node to its S and SW neighbours (setup.cu assemble_ii_kernel), so it is kept
// as a band of 2 (P+1) columns per row, for both orientations.  Per grid row
// the sweep streams B (B + 1) / 2 + B 2 (P+1) doubles per direction, against
// B (B + 1) / 2 plus the dense profile of L_{k+1,k} (about as large again) for
// a forward/backward substitution with the Cholesky factor itself.
//
// Kernel: one thread-block cluster of CS CTAs per subdomain.  A producer warp
// streams the rank's tiles (<= 32 KB each) through a ring of shared-memory
// stages with cp.async.bulk (TMA bulk copies completing on mbarriers).
//  * D^-1 phase: each consumer warp owns a contiguous run of lower tiles in
//    row-major order.  One pass over a tile (tile_pass: 8 row groups x 4 column
//    groups of lanes, every element read from shared memory once) gives the row
//    products T v_J and the column products T^T v_I; halving exchanges over
//    the lanes leave lane l with entries 2 l, 2 l + 1 of the output block.
//    Both land in per-warp register accumulators indexed by output block; the
//    warps add them into one CTA vector in warp order, which each rank pushes
//    to the owners of the rows (DSMEM).  The owner sums the ranks in order.
//  * band phase: each rank applies the band columns that fall in the rows it
//    owns and pushes the partial rows to every rank; the next phase sums the
//    ranks' partials in rank order.
// Phases are closed by data-driven signals (remote mbarrier arrivals after a
// consumer barrier), not by cluster-wide barriers; the producer is paced by
// the ring alone and runs ahead across phases.  All reductions run in a fixed
// order: results are bitwise reproducible.
// Small blocks (B <= 96) take sweep_small_kernel, very large ones (B > 1536)
// sweep_generic_kernel; both are described where they are defined.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "solver.cuh"

namespace cg = cooperative_groups;

namespace sgw {

static bool env_off(const char* name) {  // tuning / test hook: NAME=0 disables a path
  const char* e = std::getenv(name);
  return e && std::atoi(e) == 0;
}

constexpr int kSwWarps = 4;                            // consumer warps
constexpr int kSwThreads = (kSwWarps + 1) * 32;        // + one TMA producer warp
constexpr int kTileD = kTile * kTile;                  // doubles per stage
constexpr int kMaxSched = 512;                         // entries per (rank, phase type)
constexpr int kPre = 12;                               // prefetched rhs values per consumer thread
constexpr int kMaxCS = 16;                             // cluster size limit (non-portable 16)
constexpr int kSmemMax = 227 * 1024;
constexpr int kSwHeader = 512;                         // barriers, tickets, schedule heads
enum { T_SYM = 0, T_BLO = 1, T_BUP = 2, T_N = 3 };

constexpr int kMaxW = 256;                             // entries per (rank, phase type, warp)

struct SweepLayout {
  const int4* ent;     // stream entries: D^-1 tiles {off, I << 16 | J, h << 16 | wp, bytes},
                       // then A_{k+1,k} / A_{k,k+1} band chunks {off, q, 0, bytes}
  const int4* sched;   // producer stream [(rank * T_N + type) * kMaxSched + p]: {off, bytes, entry, 0}
  const int* nsched;   // [rank * T_N + type]
  const int4* wsched;  // consumer lists [((rank * T_N + type) * kSwWarps + warp) * kMaxW + p]:
                       // {stream position, first | last << 1, I << 16 | J (tile) or q (chunk), h << 16 | wp}
  const int* nwsched;  // [(rank * T_N + type) * kSwWarps + warp]
  long long blk, per_sub;  // grid-row stride; per subdomain (doubles)
  int B, H, nb, VL, NT, Rb, bw, stages;
  int slot_len, tpart_len;
  int own[kMaxCS + 1];                                  // rank r owns rows [own[r], own[r+1])
  int tlo[2][kMaxCS], thi[2][kMaxCS], toff[2][kMaxCS];  // band rows rank r contributes (LO, UP)
  int n_sym, n_ent;
  // small-block kernel (sweep_small_kernel): D_k^-1 stored full, column-major with row pitch Bp = 32 RL,
  // streamed in chunks of kSmCols columns; stage size in doubles
  int Bp, nD, stage_len, nch;
  long long lo_off, up_off;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Stage release (release semantics: this warp's shared-memory reads of the
// stage complete before the producer may overwrite it).
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// Cross-CTA phase signals: after a CTA barrier over the consumers (which
// orders every consumer thread's DSMEM pushes and earlier loads before it),
// thread r arrives with release semantics at cluster scope on rank r's
// barrier; the target's threads wait with acquire.
__device__ __forceinline__ void mbar_arrive_remote(unsigned long long* bar, int rank) {
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAITC_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra WAITC_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// split cluster barrier (release / acquire); legal for a cluster of one CTA
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait;" ::: "memory"); }
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kSwWarps * 32) : "memory");
}

// Phase order (4H - 3 phases): forward SYM_0, BLO_0, SYM_1, ..., BLO_{H-2},
// SYM_{H-1}; backward BUP_{H-2}, SYM_{H-2}, ..., BUP_0, SYM_0.
__device__ __forceinline__ void seg_info(int seg, int H, int& type, int& k, bool& fwd) {
  const int nf = 2 * H - 1;
  fwd = seg < nf;
  if (fwd) {
    k = seg >> 1;
    type = (seg & 1) ? T_BLO : T_SYM;
  } else {
    const int q = seg - nf;
    k = H - 2 - (q >> 1);
    type = (q & 1) ? T_SYM : T_BUP;
  }
}

// Swizzle of the stored tiles: element (r, c) of a tile of row stride wp sits at
// r wp + (c ^ 8 ((r >> 3) & 1)).  wp is a multiple of 16, so the XOR stays in
// the row.
__host__ __device__ __forceinline__ int sw_col(int r, int c) { return c ^ (((r >> 3) & 1) << 3); }

// One pass over a tile in shared memory gives both products.  Lane
// (rg = lane >> 2, cg = lane & 3) reads rows 8 rg + a (a < 8) and the 16-byte
// column chunks cg + 4 b (b < 8): every element is loaded once (a quarter
// warp covers two rows x four chunks, which the swizzle puts in distinct bank
// groups) and feeds the row partial rp[a] (against v_J) and, with COLS, the
// column partials cp[2 b], cp[2 b + 1] (against v_I).  Reading each tile twice
// (a row pass and a column pass) made the consumers shared-memory bound.
// Rows >= h of a stage hold stale finite data: they only reach padding rows
// (row products) or meet v_I = 0 (column products).  W > 0: full-width tile
// (constant offsets); W = 0: row stride ws < 64 (the diagonal corner tile).
template <int W, bool COLS>
__device__ __forceinline__ void tile_pass(const double* __restrict__ buf, const double* __restrict__ vj,
                                          const double* __restrict__ vi, int lane, int ws_, double (&rp)[8],
                                          double (&cp)[16]) {
  const int ws = W > 0 ? W : ws_;
  const int rg = lane >> 2, cg = lane & 3, sx = rg & 1;
  const double* base = buf + 8 * rg * ws + 2 * cg;
  double xi[8];
  if (COLS) {
#pragma unroll
    for (int a = 0; a < 8; a += 2) {
      const double2 t = *reinterpret_cast<const double2*>(vi + 8 * rg + a);
      xi[a] = t.x, xi[a + 1] = t.y;
    }
  }
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if (W == 0 && 8 * b >= ws) break;
    const double2 xj = *reinterpret_cast<const double2*>(vj + 2 * cg + 8 * b);
    const double* col = base + 8 * (b ^ sx);
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const double2 t = *reinterpret_cast<const double2*>(col + a * ws);
      rp[a] = fma(t.x, xj.x, rp[a]);
      rp[a] = fma(t.y, xj.y, rp[a]);
      if (COLS) {
        cp[2 * b] = fma(t.x, xi[a], cp[2 * b]);
        cp[2 * b + 1] = fma(t.y, xi[a], cp[2 * b + 1]);
      }
    }
  }
}

// Column partials over the 8 row groups (lane bits 2-4), halving the live
// values per step: lane ends with chunk cg + 4 rg = lane, i.e. the sums of
// columns 2 lane, 2 lane + 1 in cp[0], cp[1].  Fixed order.
__device__ __forceinline__ void reduce_cols(int lane, double (&cp)[16]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool up = lane & 16;
    const double send = up ? cp[i] : cp[i + 8], keep = up ? cp[i + 8] : cp[i];
    cp[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool up = lane & 8;
    const double send = up ? cp[i] : cp[i + 4], keep = up ? cp[i + 4] : cp[i];
    cp[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool up = lane & 4;
    const double send = up ? cp[i] : cp[i + 2], keep = up ? cp[i + 2] : cp[i];
    cp[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
}
// Row partials over the 4 column groups (lane bits 0-1): lane ends with rows
// 8 rg + 2 cg + {0, 1} = 2 lane, 2 lane + 1 in rp[0], rp[1].
__device__ __forceinline__ void reduce_rows(int lane, double (&rp)[8]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool up = lane & 2;
    const double send = up ? rp[i] : rp[i + 4], keep = up ? rp[i + 4] : rp[i];
    rp[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool up = lane & 1;
    const double send = up ? rp[i] : rp[i + 2], keep = up ? rp[i + 2] : rp[i];
    rp[i] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
  }
}

// cx[j] += a, cy[j] += b for a warp-uniform runtime j (registers stay put)
template <int NBM>
__device__ __forceinline__ void add_at(double (&cx)[NBM], double (&cy)[NBM], int j, double a, double b) {
  switch (j) {  // warp-uniform: one indirect branch instead of NBM predicated adds
#define SGW_CASE(q) \
  case q:           \
    if (q < NBM) cx[q < NBM ? q : 0] += a, cy[q < NBM ? q : 0] += b; \
    break;
    SGW_CASE(0) SGW_CASE(1) SGW_CASE(2) SGW_CASE(3) SGW_CASE(4) SGW_CASE(5) SGW_CASE(6) SGW_CASE(7)
    SGW_CASE(8) SGW_CASE(9) SGW_CASE(10) SGW_CASE(11) SGW_CASE(12) SGW_CASE(13) SGW_CASE(14) SGW_CASE(15)
    SGW_CASE(16) SGW_CASE(17) SGW_CASE(18) SGW_CASE(19) SGW_CASE(20) SGW_CASE(21) SGW_CASE(22) SGW_CASE(23)
#undef SGW_CASE
    default:
      break;
  }
}

template <int CS, int NBM>
__global__ void __launch_bounds__(kSwThreads, 1) sweep_kernel(double* __restrict__ x, const double* __restrict__ F,
                                                              const SweepLayout L) {
  extern __shared__ __align__(128) unsigned char smraw[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = CS > 1 ? (int)cluster.block_rank() : 0;
  const int s = blockIdx.x / CS;
  const int B = L.B, H = L.H, VL = L.VL, S = L.stages, nb = L.nb;
  double* stage = reinterpret_cast<double*>(smraw);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smraw + (size_t)S * kTileD * 8);
  unsigned long long* empty = full + 8;
  // ticket: stream position a stage currently holds.  Warps consume different
  // positions, so a fast warp may reach a stage a full ring ahead of the tile
  // it holds; a parity wait alone would then match the previous phase.
  volatile int* ticket = reinterpret_cast<volatile int*>(empty + 8);
  unsigned long long* slot_bar = empty + 12;   // partials of a D^-1 phase have arrived (CS > 1)
  unsigned long long* tpart_bar = empty + 13;  // band partials of a band phase have arrived (CS > 1)
  // per-phase-type schedule heads of this CTA's warps: the phase loop reads them
  // from shared memory instead of waiting on global loads at every phase start
  int4* hfirst = reinterpret_cast<int4*>(smraw + (size_t)S * kTileD * 8 + 192);  // [type][warp] first entry
  int* hnw = reinterpret_cast<int*>(smraw + (size_t)S * kTileD * 8 + 384);        // [type][warp] entries
  int* hns = hnw + T_N * kSwWarps;                                                // [type] stream length
  double* wv = reinterpret_cast<double*>(smraw + (size_t)S * kTileD * 8 + kSwHeader);  // D^-1 input (full vector)
  double* red = wv + VL;                       // CTA sum of the warps' D^-1 partials
  double* zv = CS > 1 ? red + VL : red;        // D^-1 output, owned rows
  double* slots = zv + VL;                     // [source rank][owned row] partials (CS > 1)
  double* tpart = CS > 1 ? slots + CS * L.slot_len : red + VL;  // band partials [rank segments]
  // second half of the CTA reduction tree, 16-byte aligned (double2 accesses)
  double* red2 = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(tpart + L.tpart_len) + 15) & ~uintptr_t(15));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Fs = F + (long long)s * L.per_sub;
  double* xs = x + (long long)s * H * B;
  const int nseg = 4 * H - 3;
  const int own_lo = L.own[rank], own_hi = L.own[rank + 1];

  // the ring starts zeroed: rows beyond a partial tile are then always finite
  for (int i = tid; i < S * kTileD / 2; i += kSwThreads) reinterpret_cast<double2*>(stage)[i] = make_double2(0.0, 0.0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the first bulk copy overwrites it
  if (tid < T_N * kSwWarps) {
    const int ty = tid / kSwWarps, w = tid % kSwWarps;
    hfirst[tid] = __ldg(L.wsched + (long long)((rank * T_N + ty) * kSwWarps + w) * kMaxW);
    hnw[tid] = L.nwsched[(rank * T_N + ty) * kSwWarps + w];
    if (tid < T_N) hns[tid] = L.nsched[rank * T_N + tid];
  }
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) ticket[i] = -1;
    for (int i = 0; i < S; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], 1);
    mbar_init(slot_bar, CS);
    mbar_init(tpart_bar, CS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // b_0, read before the first cluster barrier (line 0 is rewritten only at the end)
  double pre[kPre];
#pragma unroll
  for (int u = 0; u < kPre; ++u) {
    const int i = tid + u * kSwWarps * 32;
    pre[u] = (warp < kSwWarps && i < B) ? __ldcg(xs + i) : 0.0;
  }
  __syncthreads();
  cl_arrive();  // peers push into this CTA's shared memory only after it is initialised
  cl_wait();

  // --------------------------------------------------------- producer ---
  if (warp == kSwWarps) {
    unsigned pos = 0, st = 0, par = 1;  // par: parity of the release that frees stage st
    for (int seg = 0; seg < nseg; ++seg) {
      int type, k;
      bool fwd;
      seg_info(seg, H, type, k, fwd);
      const int4* sch = L.sched + (rank * T_N + type) * kMaxSched;
      const int n = L.nsched[rank * T_N + type];
      const double* base = Fs + k * L.blk;
      for (int p = 0; p < n; ++p, ++pos) {
        if (pos >= (unsigned)S) mbar_wait(&empty[st], par);
        if (lane == 0) {
          const int4 d = __ldg(sch + p);
          ticket[st] = int(pos);  // stage st now belongs to position pos (its previous tile is released)
          mbar_expect_tx(&full[st], unsigned(d.y));
          tma_bulk_load(stage + (size_t)st * kTileD, base + d.x, unsigned(d.y), &full[st]);
        }
        __syncwarp();
        if (++st == (unsigned)S) st = 0, par ^= 1u;
      }
    }
    return;  // the ring alone paces the stream: the producer runs ahead across phases
  }

  // -------------------------------------------------------- consumers ---
  unsigned pos = 0;
  unsigned sph = 0, tph = 0;  // completed phases of slot_bar / tpart_bar
  // this warp's ring cursor: stream position cgp sits in stage cst, ring lap parity cpar
  unsigned cgp = 0, cst = 0, cpar = 0;
  auto seek = [&](unsigned gp) {
    cst += gp - cgp;
    cgp = gp;
    while (cst >= (unsigned)S) cst -= S, cpar ^= 1u;
  };
  for (int seg = 0; seg < nseg; ++seg) {
    int type, k;
    bool fwd;
    seg_info(seg, H, type, k, fwd);
    const int n = hns[type];
    if (type == T_SYM) {
      // input w_k (forward: b_k minus the band partials of BLO_{k-1}; backward:
      // w_k minus those of BUP_k).  The forward stores w_k for the backward pass.
      const int t = fwd ? 0 : 1;
      const bool band_in = !(fwd && k == 0);
      if (CS > 1 && band_in) mbar_wait_cluster(tpart_bar, tph++ & 1u);
#pragma unroll
      for (int u = 0; u < kPre; ++u) {
        const int i = tid + u * kSwWarps * 32;
        if (i < VL) {
          double v = pre[u];
          if (band_in)
            for (int r = 0; r < CS; ++r)
              if (i >= L.tlo[t][r] && i < L.thi[t][r]) v -= tpart[L.toff[t][r] + i - L.tlo[t][r]];
          wv[i] = v;
          if (fwd && k > 0 && i >= own_lo && i < own_hi && i < B) xs[(long long)k * B + i] = v;
        }
      }
      // prefetch the next input: b_{k+1}, then w_{H-2} (end of the forward), w_{k-1}
      const int nxt = fwd ? (k + 1 < H ? k + 1 : H - 2) : k - 1;
      if (nxt >= 0) {
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
          const int i = tid + u * kSwWarps * 32;
          pre[u] = i < B ? __ldcg(xs + (long long)nxt * B + i) : 0.0;
        }
      }
      consumers_sync();

      double cx[NBM], cy[NBM];
#pragma unroll
      for (int q = 0; q < NBM; ++q) cx[q] = cy[q] = 0.0;
      // row partials of the current row run (rows 8 rg + a against the lane's columns)
      double rp[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      const int4* ws = L.wsched + (long long)((rank * T_N + type) * kSwWarps + warp) * kMaxW;
      const int nw = hnw[type * kSwWarps + warp];
      int4 e = hfirst[type * kSwWarps + warp];
      for (int p = 0; p < nw; ++p) {
        const int4 en = __ldg(ws + min(p + 1, nw - 1));
        const unsigned gp = pos + e.x;
        seek(gp);
        const int st = (int)cst;
        const int I = e.z >> 16, J = e.z & 0xffff, wp = e.w & 0xffff;
        const double* buf = stage + (size_t)st * kTileD;
        if (e.y & 1) {  // first tile of a row run
#pragma unroll
          for (int c = 0; c < 8; ++c) rp[c] = 0.0;
        }
        while (ticket[st] != int(gp)) {
        }
        mbar_wait(&full[st], cpar);
        double cp[16];
        if (I != J) {  // row products T v_J and column products T^T v_I from one pass
#pragma unroll
          for (int c = 0; c < 16; ++c) cp[c] = 0.0;
          tile_pass<kTile, true>(buf, wv + J * kTile, wv + I * kTile, lane, wp, rp, cp);
        } else if (wp == kTile) {
          tile_pass<kTile, false>(buf, wv + J * kTile, wv, lane, wp, rp, cp);
        } else {  // the corner tile of a grid row whose width is not a multiple of 64 (diagonal)
          tile_pass<0, false>(buf, wv + J * kTile, wv, lane, wp, rp, cp);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage
        if (I != J) {
          reduce_cols(lane, cp);
          add_at(cx, cy, J, cp[0], cp[1]);
        }
        if (e.y & 2) {  // last tile of the row run
          reduce_rows(lane, rp);
          add_at(cx, cy, I, rp[0], rp[1]);
        }
        e = en;
      }
      // CTA sum as a fixed tree (w0 + w1) + (w2 + w3): odd warps store, even
      // warps add theirs, then one pass adds the two halves; then to the owners
      static_assert(kSwWarps == 4, "the CTA reduction tree assumes four consumer warps");
      {
        double* half = (warp >> 1) ? red2 : red;
        if (warp & 1) {
#pragma unroll
          for (int q = 0; q < NBM; ++q)
            if (q < nb) reinterpret_cast<double2*>(half + q * kTile)[lane] = make_double2(cx[q], cy[q]);
        }
        consumers_sync();
        if (!(warp & 1)) {
#pragma unroll
          for (int q = 0; q < NBM; ++q)
            if (q < nb) {
              double2* dq = reinterpret_cast<double2*>(half + q * kTile) + lane;
              const double2 o = *dq;
              *dq = make_double2(cx[q] + o.x, cy[q] + o.y);
            }
        }
        consumers_sync();
      }
      if (CS > 1) {  // the two halves summed on the way to the owner of the row
        for (int i = tid; i < VL; i += kSwWarps * 32) {
          int r = 0;
          while (i >= L.own[r + 1]) ++r;
          double* dst = cluster.map_shared_rank(slots, r);
          dst[rank * L.slot_len + i - L.own[r]] = red[i] + red2[i];
        }
        consumers_sync();  // every thread's pushes precede thread 0's release
        if (tid < CS) mbar_arrive_remote(slot_bar, tid);
      } else {
        for (int i = tid; i < VL; i += kSwWarps * 32) red[i] += red2[i];
        consumers_sync();
      }
    } else {
      // input z_k / x_{k+1}: the owned rows, summed over the ranks in order
      if (CS > 1) mbar_wait_cluster(slot_bar, sph++ & 1u);
      if (CS > 1)
        for (int i = own_lo + tid; i < own_hi; i += kSwWarps * 32) {
          double v = 0.0;
          for (int r = 0; r < CS; ++r) v += slots[r * L.slot_len + i - own_lo];
          zv[i] = v;
        }
      if (!fwd)  // x_{k+1} is final
        for (int i = own_lo + tid; i < own_hi && i < B; i += kSwWarps * 32) xs[(long long)(k + 1) * B + i] = zv[i];
      consumers_sync();

      const int t = type == T_BLO ? 0 : 1, d0 = type == T_BLO ? -1 : 0;
      const int Rb = L.Rb, bw = L.bw, NT = L.NT;
      const int tl = L.tlo[t][rank], th = L.thi[t][rank], to = L.toff[t][rank];
      double* dst[CS];
#pragma unroll
      for (int r = 0; r < CS; ++r) dst[r] = CS > 1 ? cluster.map_shared_rank(tpart, r) : tpart;
      const int4* ws = L.wsched + (long long)((rank * T_N + type) * kSwWarps + warp) * kMaxW;
      const int nw = hnw[type * kSwWarps + warp];
      int4 e = hfirst[type * kSwWarps + warp];
      for (int p = 0; p < nw; ++p) {
        const int4 en = __ldg(ws + min(p + 1, nw - 1));
        const unsigned gp = pos + e.x;
        seek(gp);
        const int st = (int)cst;
        const int q = e.z;
        const double* buf = stage + (size_t)st * kTileD;
        while (ticket[st] != int(gp)) {
        }
        mbar_wait(&full[st], cpar);
        // rows lane and lane + 32 of the chunk against the owned part of their
        // column windows [c0, c0 + bw): four chains per row, fixed order
        double val[2] = {0.0, 0.0};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int r = lane + 32 * u, i = q * Rb + r;
          if (r < Rb && i < B) {
            const int c0 = (i / NT + d0) * NT;
            const int ca = max(0, own_lo - c0), cb = min(bw, own_hi - c0);
            const double* bp = buf + r;
            const double* zp = zv + c0;
            double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
            int c = ca;
            for (; c + 3 < cb; c += 4) {
              v0 = fma(bp[c * Rb], zp[c], v0);
              v1 = fma(bp[(c + 1) * Rb], zp[c + 1], v1);
              v2 = fma(bp[(c + 2) * Rb], zp[c + 2], v2);
              v3 = fma(bp[(c + 3) * Rb], zp[c + 3], v3);
            }
            for (; c < cb; ++c) v0 = fma(bp[c * Rb], zp[c], v0);
            val[u] = (v0 + v1) + (v2 + v3);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int r = lane + 32 * u, i = q * Rb + r;
          if (r < Rb && i >= tl && i < th)
#pragma unroll
            for (int rr = 0; rr < CS; ++rr) dst[rr][to + i - tl] = val[u];
        }
        e = en;
      }
      consumers_sync();  // CS > 1: every thread's pushes precede the releases below
      if (CS > 1 && tid < CS) mbar_arrive_remote(tpart_bar, tid);
    }
    pos += n;
  }
  // x_0 (the last phase was SYM_0): owned rows, ranks in order
  if (CS > 1) mbar_wait_cluster(slot_bar, sph & 1u);
  for (int i = own_lo + tid; i < own_hi && i < B; i += kSwWarps * 32) {
    double v;
    if (CS > 1) {
      v = 0.0;
      for (int r = 0; r < CS; ++r) v += slots[r * L.slot_len + i - own_lo];
    } else {
      v = red[i];
    }
    xs[i] = v;
  }
}

// ------------------------------------------------------------ storage ---
// D_k^-1 (dense column-major, lower triangle valid) -> lower tiles, diagonal
// tiles mirrored to full, swizzled by sw_col (conflict-free quarter-warp loads
// in tile_pass).
// One CTA per (subdomain, grid row, tile).
__global__ void compact_dinv_kernel(const double* __restrict__ Dinv, double* __restrict__ F, const int4* __restrict__ ent,
                                    int n_sym, long long blk, int B, int H) {
  const int e = blockIdx.x % n_sym;
  const long long sk = blockIdx.x / n_sym;  // s * H + k
  const int4 d = ent[e];
  const int I = d.y >> 16, J = d.y & 0xffff, h = d.z >> 16, wp = d.z & 0xffff;
  const double* D = Dinv + sk * (long long)B * B;
  double* out = F + sk * blk + d.x;
  for (int idx = threadIdx.x; idx < h * wp; idx += blockDim.x) {
    const int rl = idx / wp;
    const int r = I * kTile + rl, c = J * kTile + sw_col(rl, idx % wp);
    double v = 0.0;
    if (r < B && c < B) v = c <= r ? D[(long long)c * B + r] : D[(long long)r * B + c];
    out[idx] = v;
  }
}

// A_{k+1,k} (dense column-major B x B, rows: grid row k+1) -> the LO band
// (row i of grid row k+1, columns (node(i) - 1)(P+1) + c) and the UP band of
// its transpose A_{k,k+1} (row i of grid row k, columns node(i)(P+1) + c),
// chunks of Rb rows stored column-major [c][Rb].  Also records the largest
// |entry| of A_{k+1,k} outside the LO band (must be exactly zero).
__global__ void extract_band_kernel(const double* __restrict__ E, double* __restrict__ F, int B, int H, int NT, int Rb,
                                    int bw, int nch, long long blk, long long lo_off, long long up_off, int ns,
                                    unsigned long long* __restrict__ dropped) {
  const long long chunk = (long long)bw * Rb;
  const long long per = 2LL * nch * chunk;  // both bands of one (s, k)
  const long long total = (long long)ns * (H - 1) * per;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long sk = t / per;  // s * (H - 1) + k
    const long long w = t % per;
    const bool up = w >= nch * chunk;
    const long long wq = up ? w - nch * chunk : w;
    const int q = int(wq / chunk), c = int((wq % chunk) / Rb), r = int(wq % Rb);
    const int i = q * Rb + r;
    const double* A = E + sk * (long long)B * B;
    double v = 0.0;
    if (i < B) {
      const int g = (i / NT + (up ? 0 : -1)) * NT + c;
      if (g >= 0 && g < B) v = up ? A[(long long)i * B + g] : A[(long long)g * B + i];
    }
    const long long s = sk / (H - 1), k = sk % (H - 1);
    F[(s * H + k) * blk + (up ? up_off : lo_off) + wq] = v;
  }
  const long long tot2 = (long long)ns * (H - 1) * B * B;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot2; t += (long long)gridDim.x * blockDim.x) {
    const long long m = t % ((long long)B * B);
    const int c = int(m / B), r = int(m % B);
    const int g0 = (r / NT - 1) * NT;
    if (c < g0 || c >= g0 + bw) {
      const double a = fabs(E[t]);
      if (a != 0.0) atomicMax(dropped, (unsigned long long)__double_as_longlong(a));
    }
  }
}

// ------------------------------------------------- large blocks ---------
// The same block Thomas solve for interior blocks beyond the pipelined
// kernel's register-resident accumulators (B > 1536, e.g. P+1 = 91 on 32 x 32
// subdomains): one CTA per subdomain, vectors in shared memory, the D^-1 tiles
// and band chunks read straight from global memory (L2).  z = D^-1 w in two
// fixed-order passes (row products of the lower tiles, then column products
// of the strictly lower ones: every tile is read twice), so results stay
// bitwise reproducible.  Correctness path for very large PCE bases, not tuned.
constexpr int kGenThreads = 512;
__device__ void gen_dinv(const double* __restrict__ Fk, const SweepLayout& L, const double* __restrict__ w,
                         double* __restrict__ rowv, double* __restrict__ z) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kGenThreads / 32;
  // rows: warp per output row r, lanes over the columns of tiles (I, J <= I)
  for (int r = warp; r < L.B; r += nw) {
    const int I = r / kTile, rl = r % kTile;
    double acc = 0.0;
    for (int J = 0; J <= I; ++J) {
      const int4 d = L.ent[I * (I + 1) / 2 + J];
      const int wp = d.z & 0xffff;
      const double* row = Fk + d.x + (long long)rl * wp;
      for (int c = lane; c < wp; c += 32) acc = fma(__ldg(row + sw_col(rl, c)), w[J * kTile + c], acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) rowv[r] = acc;
  }
  __syncthreads();
  // columns: warp per output column c of block J, lanes over the rows of tiles (I > J, J)
  for (int col = warp; col < L.B; col += nw) {
    const int J = col / kTile, cl = col % kTile;
    double acc = 0.0;
    for (int I = J + 1; I < L.nb; ++I) {
      const int4 d = L.ent[I * (I + 1) / 2 + J];
      const int h = d.z >> 16, wp = d.z & 0xffff;
      for (int rl = lane; rl < h; rl += 32)
        acc = fma(__ldg(Fk + d.x + (long long)rl * wp + sw_col(rl, cl)), w[I * kTile + rl], acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) z[col] = rowv[col] + acc;
  }
  __syncthreads();
}
// out[i] = in[i] - sum_c band[i][c] v[g0(i) + c]  (LO: g0 = (i / NT - 1) NT, UP: (i / NT) NT)
__device__ void gen_band(const double* __restrict__ band, const SweepLayout& L, int d0, const double* __restrict__ v,
                         const double* in, double* out) {
  for (int i = threadIdx.x; i < L.B; i += kGenThreads) {
    const int q = i / L.Rb, r = i % L.Rb, g0 = (i / L.NT + d0) * L.NT;
    const double* b = band + (long long)q * L.bw * L.Rb + r;
    double acc = 0.0;
    for (int c = 0; c < L.bw; ++c) {
      const int g = g0 + c;
      if (g >= 0 && g < L.B) acc = fma(__ldg(b + (long long)c * L.Rb), v[g], acc);
    }
    out[i] = in[i] - acc;
  }
  __syncthreads();
}
__global__ void __launch_bounds__(kGenThreads, 1) sweep_generic_kernel(double* __restrict__ x, const double* __restrict__ F,
                                                                       const SweepLayout L, long long lo_off, long long up_off) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double* w = reinterpret_cast<double*>(smraw);
  double* z = w + L.VL;
  double* rowv = z + L.VL;
  const int s = blockIdx.x, B = L.B, H = L.H;
  const double* Fs = F + (long long)s * L.per_sub;
  double* xs = x + (long long)s * H * B;
  for (int i = threadIdx.x; i < L.VL; i += kGenThreads) w[i] = i < B ? xs[i] : 0.0, z[i] = 0.0;
  __syncthreads();
  for (int k = 0; k < H; ++k) {  // forward: w_k = b_k - A_{k,k-1} z_{k-1} (kept in x), z_k = D_k^-1 w_k
    if (k > 0) {
      for (int i = threadIdx.x; i < B; i += kGenThreads) rowv[i] = xs[(long long)k * B + i];
      __syncthreads();
      gen_band(Fs + (long long)(k - 1) * L.blk + lo_off, L, -1, z, rowv, w);
      for (int i = threadIdx.x; i < B; i += kGenThreads) xs[(long long)k * B + i] = w[i];
    }
    gen_dinv(Fs + (long long)k * L.blk, L, w, rowv, z);
  }
  for (int i = threadIdx.x; i < B; i += kGenThreads) xs[(long long)(H - 1) * B + i] = z[i];
  for (int k = H - 2; k >= 0; --k) {  // backward: x_k = D_k^-1 (w_k - A_{k,k+1} x_{k+1})
    for (int i = threadIdx.x; i < B; i += kGenThreads) rowv[i] = xs[(long long)k * B + i];
    __syncthreads();
    gen_band(Fs + (long long)k * L.blk + up_off, L, 0, z, rowv, w);
    gen_dinv(Fs + (long long)k * L.blk, L, w, rowv, z);
    for (int i = threadIdx.x; i < B; i += kGenThreads) xs[(long long)k * B + i] = z[i];
    __syncthreads();
  }
}

// ------------------------------------------------- small blocks ---------
// The same block Thomas solve for small interior blocks (B <= 96: few PCE
// terms or small subdomains, e.g. C1 with B = 90 or deterministic solves with
// B = W).  There the tiled kernel is bound by its CTA barriers and cluster
// handshakes (about 2 us per phase, 4 phases per grid row), not by bytes.
// Here one OWNER warp holds a subdomain's vectors in registers: lane l has
// rows l, l + 32, l + 64, so the chain w_k -> z_k = D_k^-1 w_k -> band
// product -> w_{k+1} stays in one warp.  Three helper warps share the D^-1
// product (each consumer warp takes 4 of a chunk's 16 columns; the owner adds
// the partials in warp order), which costs two named barriers per grid row.
// D_k^-1 is stored full (symmetric: column c of the stored block is row c),
// column-major with row pitch Bp = 32 RL: lane l reads element (l + 32 u, c),
// i.e. consecutive addresses, against the broadcast w[c].  A producer warp
// streams chunks of kSmCols columns and the band chunks through a ring of TMA
// bulk copies; the bands use the tiled kernel's chunk format (Rb = 64 rows, so
// a chunk's rows lane, lane + 32 are rows the owner lane holds: u = 2 q,
// 2 q + 1).  Fixed summation order: bitwise reproducible.
constexpr int kSmCols = 16;     // D^-1 columns per stage
constexpr int kSmMaxStages = 16;
constexpr int kSmCons = 4;      // consumer warps (owner + helpers)
constexpr int kSmThreads = 32 * (kSmCons + 1);
__device__ __forceinline__ void small_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kSmCons * 32) : "memory"); }

template <int RL>
__global__ void __launch_bounds__(kSmThreads, 1) sweep_small_kernel(double* __restrict__ x, const double* __restrict__ F,
                                                                    const SweepLayout L) {
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int Bp = 32 * RL;
  const int s = blockIdx.x, B = L.B, H = L.H, S = L.stages;
  double* stage = reinterpret_cast<double*>(smraw);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smraw + (size_t)S * L.stage_len * 8);
  unsigned long long* empty = full + kSmMaxStages;
  double* wv = reinterpret_cast<double*>(empty + kSmMaxStages);  // D^-1 input [Bp], broadcast to the lanes
  double* zv = wv + Bp;              // D^-1 output [32 | Bp | 32]: zero guards of >= NT entries on both sides
  double* zpart = zv + Bp + 64;      // helpers' partial products [kSmCons - 1][Bp]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Fs = F + (long long)s * L.per_sub;
  double* xs = x + (long long)s * H * B;
  const int nseg = 4 * H - 3;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], kSmCons);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 2 * Bp + 64; i += kSmThreads) wv[i] = 0.0;  // wv and zv with its guards
  __syncthreads();

  if (warp == kSmCons) {  // ------------------------------------ producer ---
    unsigned pos = 0, st = 0, par = 1;
    for (int seg = 0; seg < nseg; ++seg) {
      int type, k;
      bool fwd;
      seg_info(seg, H, type, k, fwd);
      const double* base = Fs + k * L.blk + (type == T_SYM ? 0 : type == T_BLO ? L.lo_off : L.up_off);
      const int n = type == T_SYM ? L.nD : L.nch;
      const int len = type == T_SYM ? kSmCols * Bp : L.bw * L.Rb;
      for (int p = 0; p < n; ++p, ++pos) {
        if (pos >= (unsigned)S) mbar_wait(&empty[st], par);
        if (lane == 0) {
          mbar_expect_tx(&full[st], unsigned(len * 8));
          tma_bulk_load(stage + (size_t)st * L.stage_len, base + (long long)p * len, unsigned(len * 8), &full[st]);
        }
        __syncwarp();
        if (++st == (unsigned)S) st = 0, par ^= 1u;
      }
    }
    return;
  }

  // ----------------------------------------------------------- consumers ---
  const int NT = L.NT, bw = L.bw, Rb = L.Rb;
  const bool owner = warp == 0;
  unsigned st = 0, par = 0;
  auto next_stage = [&]() {
    if (++st == (unsigned)S) st = 0, par ^= 1u;
  };
  double pre[RL], z[RL], t[RL];
#pragma unroll
  for (int u = 0; u < RL; ++u) {
    const int r = lane + 32 * u;
    pre[u] = owner && r < B ? __ldcg(xs + r) : 0.0;
    z[u] = t[u] = 0.0;
  }
  double* zc = zv + 32;  // zc[-NT .. B + NT) is addressable; entries outside [0, B) stay zero
  int node0[RL];         // first column of row lane + 32 u's own node (band windows start at node0 - NT / node0)
#pragma unroll
  for (int u = 0; u < RL; ++u) node0[u] = (lane + 32 * u) / NT * NT;
  for (int seg = 0; seg < nseg; ++seg) {
    int type, k;
    bool fwd;
    seg_info(seg, H, type, k, fwd);
    if (type == T_SYM) {
      if (owner) {
        // w_k = b_k - (band partial of the previous phase); the forward stores it for the backward pass
        const bool band_in = !(fwd && k == 0);
#pragma unroll
        for (int u = 0; u < RL; ++u) {
          const int r = lane + 32 * u;
          const double w = band_in ? pre[u] - t[u] : pre[u];
          wv[r] = w;
          if (fwd && k > 0 && r < B) xs[(long long)k * B + r] = w;
        }
        const int nxt = fwd ? (k + 1 < H ? k + 1 : H - 2) : k - 1;
        if (nxt >= 0) {
#pragma unroll
          for (int u = 0; u < RL; ++u) {
            const int r = lane + 32 * u;
            pre[u] = r < B ? __ldcg(xs + (long long)nxt * B + r) : 0.0;
          }
        }
      }
      small_sync();  // w_k is in wv (and the owner has read the helpers' previous partials)
      double za[RL], zb[RL];
#pragma unroll
      for (int u = 0; u < RL; ++u) za[u] = zb[u] = 0.0;
      for (int q = 0; q < L.nD; ++q) {
        // this warp's 4 of the chunk's 16 columns (columns past B are stored zeros and meet w = 0)
        const double* buf = stage + (size_t)st * L.stage_len + 4 * warp * Bp + lane;
        const double* wq = wv + q * kSmCols + 4 * warp;
        mbar_wait(&full[st], par);
        const double2 w01 = *reinterpret_cast<const double2*>(wq);
        const double2 w23 = *reinterpret_cast<const double2*>(wq + 2);
#pragma unroll
        for (int u = 0; u < RL; ++u) {
          za[u] = fma(buf[32 * u], w01.x, za[u]);
          zb[u] = fma(buf[Bp + 32 * u], w01.y, zb[u]);
          za[u] = fma(buf[2 * Bp + 32 * u], w23.x, za[u]);
          zb[u] = fma(buf[3 * Bp + 32 * u], w23.y, zb[u]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        next_stage();
      }
      if (!owner) {
#pragma unroll
        for (int u = 0; u < RL; ++u) zpart[(warp - 1) * Bp + lane + 32 * u] = za[u] + zb[u];
      }
      small_sync();  // the helpers' partials are in zpart
      if (owner) {
#pragma unroll
        for (int u = 0; u < RL; ++u) {
          const int r = lane + 32 * u;
          double v = za[u] + zb[u];
#pragma unroll
          for (int h = 0; h < kSmCons - 1; ++h) v += zpart[h * Bp + r];
          z[u] = v;
          if (r < B) zc[r] = v;
        }
        __syncwarp();
      }
    } else {
      if (!owner) {  // helpers only release the band stages (the owner reads them)
        for (int q = 0; q < L.nch; ++q) {
          if (lane == 0) mbar_arrive(&empty[st]);
          next_stage();
        }
        continue;
      }
      // x_{k+1} is final in the backward pass
      if (!fwd) {
#pragma unroll
        for (int u = 0; u < RL; ++u) {
          const int r = lane + 32 * u;
          if (r < B) xs[(long long)(k + 1) * B + r] = z[u];
        }
      }
      const int d0 = type == T_BLO ? -1 : 0;
#pragma unroll
      for (int u = 0; u < RL; ++u) t[u] = 0.0;
      for (int q = 0; q < L.nch; ++q) {
        const double* buf = stage + (size_t)st * L.stage_len;
        mbar_wait(&full[st], par);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int u = 2 * q + h;  // chunk rows lane, lane + 32 = rows lane + 32 u of the block
          const int r = lane + 32 * h, i = q * Rb + r;
          if (u < RL && i < B) {
            int c0 = 0;  // window [c0, c0 + bw): zc is zero outside [0, B)
#pragma unroll
            for (int uu = 0; uu < RL; ++uu)
              if (uu == u) c0 = node0[uu] + d0 * NT;
            const double* bp = buf + r;
            const double* zp = zc + c0;
            double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
            int c = 0;
            for (; c + 3 < bw; c += 4) {
              v0 = fma(bp[c * Rb], zp[c], v0);
              v1 = fma(bp[(c + 1) * Rb], zp[c + 1], v1);
              v2 = fma(bp[(c + 2) * Rb], zp[c + 2], v2);
              v3 = fma(bp[(c + 3) * Rb], zp[c + 3], v3);
            }
            for (; c < bw; ++c) v0 = fma(bp[c * Rb], zp[c], v0);
            const double val = (v0 + v1) + (v2 + v3);
#pragma unroll
            for (int uu = 0; uu < RL; ++uu)
              if (uu == u) t[uu] = val;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        next_stage();
      }
    }
  }
  // x_0 (the last phase was SYM_0)
  if (owner) {
#pragma unroll
    for (int u = 0; u < RL; ++u) {
      const int r = lane + 32 * u;
      if (r < B) xs[r] = z[u];
    }
  }
}

// D_k^-1 (dense column-major, lower triangle valid) -> the small kernel's
// full column-major block of nD kSmCols columns with row pitch Bp (zeros
// past B).  One CTA per (subdomain, grid row).
__global__ void compact_dinv_small_kernel(const double* __restrict__ Dinv, double* __restrict__ F, long long blk, int B,
                                          int Bp, int ncol) {
  const long long sk = blockIdx.x;
  const double* D = Dinv + sk * (long long)B * B;
  double* out = F + sk * blk;
  for (int idx = threadIdx.x; idx < ncol * Bp; idx += blockDim.x) {
    const int c = idx / Bp, r = idx % Bp;
    double v = 0.0;
    if (r < B && c < B) v = c <= r ? D[(long long)c * B + r] : D[(long long)r * B + c];
    out[idx] = v;
  }
}

using SweepFn = void (*)(double*, const double*, const SweepLayout);
static SweepFn sweep_fn(int cs, int nbm) {
#define SGW_SW(C)                                                  \
  case C:                                                          \
    return nbm == 12 ? (SweepFn)sweep_kernel<C, 12> : (SweepFn)sweep_kernel<C, 24>;
  switch (cs) {
    SGW_SW(1)
    SGW_SW(2)
    SGW_SW(4)
    SGW_SW(8)
    default:
      return nbm == 12 ? (SweepFn)sweep_kernel<16, 12> : (SweepFn)sweep_kernel<16, 24>;
  }
#undef SGW_SW
}

static size_t smem_bytes(int stages, int VL, int CS, int slot_len, int tpart_len) {
  const size_t vec = 3 * (size_t)VL + (CS > 1 ? (size_t)VL + (size_t)CS * slot_len : 0) + (size_t)tpart_len + 2;
  return (size_t)stages * kTileD * 8 + kSwHeader + vec * 8;
}

void GpuSolver::build_sweep_layout() {
  const int H = G.H, nb = (B + kTile - 1) / kTile, VL = nb * kTile;
  const int bw = 2 * NT;
  int Rb = 64;
  while (Rb > 16 && Rb * bw > kTileD) Rb /= 2;
  // blocks beyond the pipelined kernel's limits: the large-block kernel
  sweep_generic_ = B > kPre * kSwWarps * 32 || Rb * bw > kTileD || std::getenv("SGW_SWEEP_GENERIC") != nullptr;
  if (sweep_generic_ && 3 * (size_t)VL * 8 > (size_t)kSmemMax)
    throw Error(1, "interior block too large for the sweep kernels (3 B doubles of shared memory)");
  const int nch = (B + Rb - 1) / Rb;
  auto hgt = [&](int I) { return std::min(kTile, B - I * kTile); };
  // stored tile width: a multiple of 16 so that the swizzle (column pairs
  // XOR 2 (row & 7)) stays inside the row and both products are conflict-free
  auto wpad = [&](int J) { return (std::min(kTile, B - J * kTile) + 15) & ~15; };
  std::vector<int4> ent;
  long long off = 0;
  for (int I = 0; I < nb; ++I)
    for (int J = 0; J <= I; ++J) {
      ent.push_back(make_int4((int)off, I << 16 | J, hgt(I) << 16 | wpad(J), hgt(I) * wpad(J) * 8));
      off += (long long)hgt(I) * wpad(J);
    }
  const int n_sym = (int)ent.size();
  const long long lo_off = (off + 31) & ~31LL;  // 256-byte aligned
  const long long up_off = (lo_off + (long long)nch * bw * Rb + 31) & ~31LL;
  for (int band = 0; band < 2; ++band)
    for (int q = 0; q < nch; ++q)
      ent.push_back(make_int4(int((band ? up_off : lo_off) + (long long)q * bw * Rb), q, 0, bw * Rb * 8));
  const long long blk = (up_off + (long long)nch * bw * Rb + 31) & ~31LL;
  if (blk >= (1LL << 31)) throw Error(1, "interior block too large for the sweep layout");

  if (sweep_generic_) {
    SweepLayout L{};
    std::vector<int> raw(ent.size() * 4);
    std::memcpy(raw.data(), ent.data(), raw.size() * sizeof(int));
    sw_off.upload(raw);
    L.ent = reinterpret_cast<const int4*>(sw_off.p);
    L.blk = blk, L.per_sub = (long long)H * blk;
    L.B = B, L.H = H, L.nb = nb, L.VL = VL, L.NT = NT, L.Rb = Rb, L.bw = bw;
    L.n_sym = n_sym, L.n_ent = (int)ent.size();
    delete sweep_layout_;
    sweep_layout_ = new SweepLayout(L);
    sweep_lo_off_ = lo_off, sweep_up_off_ = up_off, sweep_nch_ = nch, sweep_cs_ = 1;
    Fcomp.alloc(size_t(NS) * L.per_sub);
    ensure_dyn_smem((const void*)sweep_generic_kernel, 3 * (size_t)VL * 8);
    return;
  }
  // small blocks: one consumer warp per subdomain (sweep_small_kernel)
  // (SGW_SWEEP_CS, the test hook that forces a cluster size, asks for the tiled kernel)
  sweep_small_ = B <= 96 && Rb == 64 && NT <= 32 && !env_off("SGW_SWEEP_SMALL") && !std::getenv("SGW_SWEEP_CS");
  if (sweep_small_) {
    SweepLayout L{};
    const int RL = (B + 31) / 32, Bp = 32 * RL, nD = (B + kSmCols - 1) / kSmCols;
    const long long lo = ((long long)nD * kSmCols * Bp + 31) & ~31LL;
    const long long up = (lo + (long long)nch * bw * Rb + 31) & ~31LL;
    L.blk = (up + (long long)nch * bw * Rb + 31) & ~31LL;
    L.per_sub = (long long)H * L.blk;
    L.B = B, L.H = H, L.nb = nb, L.VL = VL, L.NT = NT, L.Rb = Rb, L.bw = bw;
    L.Bp = Bp, L.nD = nD, L.nch = nch, L.lo_off = lo, L.up_off = up;
    L.stage_len = std::max(kSmCols * Bp, bw * Rb);
    L.stages = std::max(2, std::min<int>(kSmMaxStages, int((200 * 1024) / (L.stage_len * 8))));
    delete sweep_layout_;
    sweep_layout_ = new SweepLayout(L);
    sweep_lo_off_ = lo, sweep_up_off_ = up, sweep_nch_ = nch, sweep_cs_ = 1;
    Fcomp.alloc(size_t(NS) * L.per_sub);
    const void* fn = RL == 1 ? (const void*)sweep_small_kernel<1> : RL == 2 ? (const void*)sweep_small_kernel<2>
                                                                             : (const void*)sweep_small_kernel<3>;
    ensure_dyn_smem(fn, sweep_smem_bytes());
    return;
  }
  // cluster size: about one wave of CTAs over the 148 SMs
  int CS = NS >= 100 ? 1 : NS >= 48 ? 2 : NS >= 24 ? 4 : NS >= 12 ? 8 : 16;
  // small blocks (C1: B = 90, two tile rows) gain nothing from more CTAs than
  // about half their tile rows, and every rank adds cluster traffic per phase
  while (CS > 1 && CS > nb / 2) CS /= 2;
  if (const char* e = std::getenv("SGW_SWEEP_CS")) {  // test hook: force a cluster size
    const int v = std::atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) CS = v;
  }
  const int nbm = nb <= 12 ? 12 : 24;
  SweepLayout L{};
  auto plan = [&](int cs) {
    // row ownership: contiguous 64-row blocks
    for (int r = 0; r <= cs; ++r) L.own[r] = r == cs ? VL : kTile * (r * nb / cs);
    L.slot_len = 0;
    for (int r = 0; r < cs; ++r) L.slot_len = std::max(L.slot_len, L.own[r + 1] - L.own[r]);
    // band rows each rank contributes to: rows whose column window meets its rows
    L.tpart_len = 0;
    for (int t = 0; t < 2; ++t) {
      int acc = 0;
      for (int r = 0; r < cs; ++r) {
        int lo = B, hi = 0;
        const int a = L.own[r], b = std::min(L.own[r + 1], B);
        for (int i = 0; i < B && a < b; ++i) {
          const int g = (i / NT + (t ? 0 : -1)) * NT;
          if (g < b && g + bw > a) lo = std::min(lo, i), hi = std::max(hi, i + 1);
        }
        if (lo >= hi) lo = hi = 0;
        L.tlo[t][r] = lo, L.thi[t][r] = hi, L.toff[t][r] = acc;
        acc += hi - lo;
      }
      L.tpart_len = std::max(L.tpart_len, acc);
    }
    int st = 6;
    while (st > 3 && smem_bytes(st, VL, cs, L.slot_len, L.tpart_len) > (size_t)kSmemMax) --st;
    L.stages = st;
  };
  plan(CS);
  if (CS == 16) {  // non-portable cluster size: only if 16-CTA clusters of this size are schedulable
    const size_t smem = smem_bytes(L.stages, VL, 16, L.slot_len, L.tpart_len);
    const void* fn = (const void*)sweep_fn(16, nbm);
    int nclus = 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16), cfg.blockDim = dim3(kSwThreads), cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16, attr[0].val.clusterDim.y = 1, attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr, cfg.numAttrs = 1;
    if (smem > (size_t)kSmemMax || cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        (ensure_dyn_smem(fn, smem), false) ||
        cudaOccupancyMaxActiveClusters(&nclus, fn, &cfg) != cudaSuccess || nclus < NS) {
      (void)cudaGetLastError();
      CS = 8;
      plan(CS);
    }
  }
  if (smem_bytes(L.stages, VL, CS, L.slot_len, L.tpart_len) > (size_t)kSmemMax)
    throw Error(1, "interior block too large for the sweep kernel's shared memory");
  sweep_cs_ = CS;

  // schedules.  D^-1: the lower tiles in row-major order, cut into CS x 4
  // contiguous runs of equal work (rank-major; an off-diagonal tile costs a
  // row and a column product, a diagonal one a row product); a rank streams its
  // warps' tiles interleaved.  Bands: the chunks holding the rank's rows, dealt
  // to the warps in turn.
  const int nbin = CS * kSwWarps;
  std::vector<int4> sched((size_t)CS * T_N * kMaxSched, make_int4(0, 0, 0, 0));
  std::vector<int> nsched((size_t)CS * T_N, 0);
  std::vector<int4> wsched((size_t)CS * T_N * kSwWarps * kMaxW, make_int4(0, 0, 0, 0));
  std::vector<int> nwsched((size_t)CS * T_N * kSwWarps, 0);
  auto push = [&](int q, int t, int w, int e, int flags, int key) {
    int& n = nsched[q * T_N + t];
    int& nw = nwsched[(q * T_N + t) * kSwWarps + w];
    if (n >= kMaxSched || nw >= kMaxW) throw Error(1, "sweep: schedule too long");
    sched[(size_t)(q * T_N + t) * kMaxSched + n] = make_int4(ent[e].x, ent[e].w, e, 0);
    wsched[((size_t)(q * T_N + t) * kSwWarps + w) * kMaxW + nw] = make_int4(n, flags, key, ent[e].z);
    ++n, ++nw;
  };
  {
    std::vector<double> wt(n_sym);
    double total = 0.0;
    for (int e = 0; e < n_sym; ++e) {
      const int I = ent[e].y >> 16, J = ent[e].y & 0xffff;
      wt[e] = (I == J ? 1.0 : 2.0) * (ent[e].z >> 16), total += wt[e];
    }
    std::vector<std::vector<int>> bins(nbin);
    double acc = 0.0;
    int b = 0;
    for (int e = 0; e < n_sym; ++e) {
      while (b < nbin - 1 && acc + 0.5 * wt[e] > (b + 1) * total / nbin) ++b;
      bins[b].push_back(e);
      acc += wt[e];
    }
    for (int q = 0; q < CS; ++q)
      for (size_t i = 0;; ++i) {
        bool any = false;
        for (int w = 0; w < kSwWarps; ++w) {
          const auto& tl = bins[q * kSwWarps + w];
          if (i >= tl.size()) continue;
          const int I = ent[tl[i]].y >> 16;
          const bool first = i == 0 || (ent[tl[i - 1]].y >> 16) != I;
          const bool last = i + 1 == tl.size() || (ent[tl[i + 1]].y >> 16) != I;
          push(q, T_SYM, w, tl[i], int(first) | int(last) << 1, ent[tl[i]].y);
          any = true;
        }
        if (!any) break;
      }
  }
  for (int t = 0; t < 2; ++t)
    for (int q = 0; q < CS; ++q)
      if (L.thi[t][q] > L.tlo[t][q])
        for (int c = L.tlo[t][q] / Rb, i = 0; c <= (L.thi[t][q] - 1) / Rb; ++c, ++i)
          push(q, T_BLO + t, i % kSwWarps, n_sym + t * nch + c, 0, c);
  std::vector<int> raw(ent.size() * 4), sraw(sched.size() * 4), wraw(wsched.size() * 4);
  std::memcpy(raw.data(), ent.data(), raw.size() * sizeof(int));
  std::memcpy(sraw.data(), sched.data(), sraw.size() * sizeof(int));
  std::memcpy(wraw.data(), wsched.data(), wraw.size() * sizeof(int));
  sw_off.upload(raw);
  sw_cuts.upload(sraw);
  sw_ncut.upload(nsched);
  sw_wcuts.upload(wraw);
  sw_nw.upload(nwsched);
  L.wsched = reinterpret_cast<const int4*>(sw_wcuts.p);
  L.nwsched = sw_nw.p;
  L.ent = reinterpret_cast<const int4*>(sw_off.p);
  L.sched = reinterpret_cast<const int4*>(sw_cuts.p);
  L.nsched = sw_ncut.p;
  L.blk = blk, L.per_sub = (long long)H * blk;
  L.B = B, L.H = H, L.nb = nb, L.VL = VL, L.NT = NT, L.Rb = Rb, L.bw = bw;
  if (const char* e = std::getenv("SGW_SWEEP_STAGES"))  // tuning hook
    L.stages = std::max(2, std::min(L.stages, std::atoi(e)));
  L.n_sym = n_sym, L.n_ent = (int)ent.size();
  delete sweep_layout_;
  sweep_layout_ = new SweepLayout(L);
  sweep_lo_off_ = lo_off, sweep_up_off_ = up_off, sweep_nch_ = nch, sweep_nbm_ = nbm;
  Fcomp.alloc(size_t(NS) * L.per_sub);
  const size_t smem = sweep_smem_bytes();
  const void* fn = (const void*)sweep_fn(CS, nbm);
  ensure_dyn_smem(fn, smem);
  if (CS == 16) SGW_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

// A_{k+1,k} blocks of subdomains [b0, b0 + nb) (batch-local Lsub, before the
// factorization overwrites them) -> the band chunks in Fcomp
void GpuSolver::extract_band_batch(int b0, int nb) {
  const SweepLayout& L = *sweep_layout_;
  if (L.H < 2) return;
  DBuf<unsigned long long> drop;
  drop.alloc(1);
  drop.zero(st_);
  extract_band_kernel<<<8 * kNumSMs * 4, 256, 0, st_>>>(Lsub.p, Fcomp.p + (size_t)b0 * L.per_sub, L.B, L.H, L.NT, L.Rb,
                                                        L.bw, sweep_nch_, L.blk, sweep_lo_off_, sweep_up_off_, nb,
                                                        drop.p);
  SGW_LAUNCHED();
  unsigned long long h = 0;
  SGW_CUDA(cudaMemcpyAsync(&h, drop.p, sizeof(h), cudaMemcpyDeviceToHost, st_));
  SGW_CUDA(cudaStreamSynchronize(st_));
  if (h != 0) {
    double v;
    std::memcpy(&v, &h, sizeof(v));
    throw Error(2, "interior operator: grid-row coupling outside the S/SW band (" + std::to_string(v) + ")");
  }
}

// D_k^-1 blocks of subdomains [b0, b0 + nb) (batch-local, dense) -> tiles
void GpuSolver::compact_dinv_batch(int b0, int nb, const double* dinv) {
  const SweepLayout& L = *sweep_layout_;
  if (sweep_small_) {
    compact_dinv_small_kernel<<<(unsigned)((long long)nb * L.H), 256, 0, st_>>>(dinv, Fcomp.p + (size_t)b0 * L.per_sub, L.blk,
                                                                                L.B, L.Bp, L.nD * kSmCols);
    SGW_LAUNCHED();
    return;
  }
  const long long nblk = (long long)nb * L.H * L.n_sym;
  if (nblk >= (1LL << 31)) throw Error(1, "sweep: too many tiles per setup batch");
  compact_dinv_kernel<<<(unsigned)nblk, 256, 0, st_>>>(dinv, Fcomp.p + (size_t)b0 * L.per_sub, L.ent, L.n_sym, L.blk,
                                                       L.B, L.H);
  SGW_LAUNCHED();
}

void destroy_sweep_layout(SweepLayout* p) { delete p; }

size_t GpuSolver::sweep_smem_bytes() const {
  const SweepLayout& L = *sweep_layout_;
  if (sweep_generic_) return 3 * (size_t)L.VL * 8;
  if (sweep_small_)
    return (size_t)L.stages * L.stage_len * 8 + 2 * kSmMaxStages * 8 + (size_t)((2 + kSmCons - 1) * L.Bp + 64) * 8;
  return smem_bytes(L.stages, L.VL, sweep_cs_, L.slot_len, L.tpart_len);
}

void GpuSolver::sweep(double* x) {
  const SweepLayout& L = *sweep_layout_;
  cudaEvent_t e0;
  KP.begin(K_SWEEP, st_, &e0);
  if (sweep_generic_) {
    sweep_generic_kernel<<<NS, kGenThreads, sweep_smem_bytes(), st_>>>(x, Fcomp.p, L, sweep_lo_off_, sweep_up_off_);
    SGW_LAUNCHED();
    KP.end(st_);
    return;
  }
  if (sweep_small_) {
    const int RL = (L.B + 31) / 32;
    const size_t smem = sweep_smem_bytes();
    if (RL == 1) sweep_small_kernel<1><<<NS, kSmThreads, smem, st_>>>(x, Fcomp.p, L);
    else if (RL == 2) sweep_small_kernel<2><<<NS, kSmThreads, smem, st_>>>(x, Fcomp.p, L);
    else sweep_small_kernel<3><<<NS, kSmThreads, smem, st_>>>(x, Fcomp.p, L);
    SGW_LAUNCHED();
    KP.end(st_);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(NS * sweep_cs_);
  cfg.blockDim = dim3(kSwThreads);
  cfg.dynamicSmemBytes = sweep_smem_bytes();
  cfg.stream = st_;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = sweep_cs_;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const double* F = Fcomp.p;
  SGW_CUDA(cudaLaunchKernelEx(&cfg, sweep_fn(sweep_cs_, sweep_nbm_), x, F, L));
  SGW_LAUNCHED();
  KP.end(st_);
}

// Algorithmic bytes of one forward + backward solve: D_k^-1 (unique entries)
// once per grid row and direction except the shared last row (2H - 1 applies),
// and the nonzero band of A_{k+1,k} once per direction (the first / last node
// of a row has one neighbour node in the window).
double GpuSolver::bytes_sweep() const {
  const SweepLayout& L = *sweep_layout_;
  const double dinv = 0.5 * double(L.B) * (L.B + 1);
  const double band = double(L.B) * L.bw - double(NT) * NT;
  return 8.0 * double(NS) * (double(2 * L.H - 1) * dinv + 2.0 * double(L.H - 1) * band);
}

}  // namespace sgw
