// Batched interior Dirichlet solve x <- A_II^-1 x for every subdomain
// (src/sg.cpp:317 and :350: SimplicialLLT::solve, restated block-wise).
//
// A_II = L L^T is block lower-bidiagonal over the H interior grid rows
// (blocks B = W (P+1), node-major / term-minor):
//   forward   y_k = L_kk^-1 (b_k - L_{k,k-1} y_{k-1})
//   backward  x_k = L_kk^-T (y_k - L_{k+1,k}^T x_{k+1})
// Both products of a block row are stored as 64 x 64 tiles (row-major, width
// padded to even, zeros outside the factor's profile):
//   INV_k = L_kk^-1     tiles (I, J), J <= I
//   SUB_k = L_{k+1,k}   tiles (I, J), J >= Jmin(I): row r of L_{k+1,k} is zero left of
//                       column c0(r) = ((node(r) - 1)(P+1)), so whole tiles vanish
// The forward sweep multiplies the tiles (row sums); the backward sweep
// multiplies their transposes from the same storage (column sums), so the
// factor is held once.
//
// Kernel: one thread-block cluster of CS CTAs per subdomain.  Every output
// block (64 rows of a forward product, 64 columns of a backward one) belongs
// to one consumer warp of one rank, which accumulates the block's tiles in
// registers: lane l owns tile columns 2l, 2l+1, so a forward block needs one
// 64-to-2 butterfly reduction at its end and a backward block none.  A
// producer warp streams the rank's tiles (32 KB each) through a ring of
// shared-memory stages with cp.async.bulk (TMA bulk copies completing on
// mbarriers), interleaving the warps' tiles and running ahead across block
// rows.  Results are pushed into every rank's copy of the vector through
// DSMEM; one split cluster barrier closes each block-row phase.  Reductions
// run in a fixed order: results are bitwise reproducible.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "solver.cuh"

namespace cg = cooperative_groups;

namespace sgw {

constexpr int kSwWarps = 4;                        // consumer warps
constexpr int kSwThreads = (kSwWarps + 1) * 32;    // + one TMA producer warp
constexpr int kTileD = kTile * kTile;              // doubles per stage (one tile)
constexpr int kMaxSched = 512;                     // tiles per (rank, product)
constexpr int kPre = 12;                           // prefetched rhs values per consumer thread
enum { T_INV = 0, T_SUB = 1, T_INVT = 2, T_SUBT = 3, T_N = 4 };

struct SweepLayout {
  const int4* tiles[2];  // INV / SUB tile tables: {offset, I << 16 | J, h << 16 | wp, 0}
  const int4* sched;     // [(rank * T_N + type) * kMaxSched + p]: {tile, warp | first << 8 | last << 9, block, 0}
  const int* nsched;     // [rank * T_N + type]
  long long sub_off, blk, per_sub;  // SUB tiles inside a block row; block-row stride; per subdomain
  int B, H, nb, VL, stages;
  int n_inv, n_all;  // tile-table sizes (host side: compaction)
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
// split cluster barrier (release / acquire); legal for a cluster of one CTA
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait;" ::: "memory"); }
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kSwWarps * 32) : "memory");
}

// Streaming order: forward INV_0, SUB_0, INV_1, ..., INV_{H-1}; backward
// INVT_{H-1}, SUBT_{H-2}, INVT_{H-2}, ..., INVT_0 (SUB_k / SUBT_k hold L_{k+1,k}).
__device__ __forceinline__ void seg_info(int seg, int H, int& type, int& k, bool& fwd) {
  const int nf = 2 * H - 1;
  fwd = seg < nf;
  const int q = fwd ? seg : seg - nf;
  const int j = (q + 1) >> 1;
  const bool sub = q & 1;
  type = fwd ? (sub ? T_SUB : T_INV) : (sub ? T_SUBT : T_INVT);
  k = fwd ? (sub ? j - 1 : j) : H - 1 - j;
}

// 64 lane partials (rows 0..63 of a block, this lane's two columns) -> sums
// of rows 2 lane and 2 lane + 1 in a[0], a[1]: a butterfly that halves the
// live values at every level (62 exchanges for 64 rows).
__device__ __forceinline__ void butterfly64(double (&a)[kTile], int lane) {
#pragma unroll
  for (int lvl = 0; lvl < 5; ++lvl) {
    const int half = 32 >> lvl, m = 16 >> lvl;
    const bool up = lane & m;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = up ? a[i] : a[i + half], keep = up ? a[i + half] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
}

template <int CS>
__global__ void __launch_bounds__(kSwThreads, 1) sweep_kernel(double* __restrict__ x, const double* __restrict__ F,
                                                              SweepLayout L) {
  extern __shared__ __align__(128) unsigned char smraw[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = CS > 1 ? (int)cluster.block_rank() : 0;
  const int s = blockIdx.x / CS;
  const int B = L.B, H = L.H, VL = L.VL, S = L.stages;
  double* stage = reinterpret_cast<double*>(smraw);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smraw + (size_t)S * kTileD * 8);
  unsigned long long* empty = full + 8;
  // ticket: stream position a stage currently holds.  Warps consume different
  // positions, so a fast warp may reach a stage a full ring ahead of the tile
  // it holds; a parity wait alone would then match the previous phase.
  volatile int* ticket = reinterpret_cast<volatile int*>(empty + 8);
  double* vv = reinterpret_cast<double*>(empty + 12);  // y_k (forward) / s_k (backward), zero padded to VL
  double* tv = vv + VL;                                 // t_k (forward) / x_k (backward)
  double* bv = tv + VL;                                 // right-hand side block: b_{k+1} / y_k
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Fs = F + (long long)s * L.per_sub;
  double* xs = x + (long long)s * H * B;
  const int nseg = 2 * (2 * H - 1);

  for (int i = tid; i < 3 * VL; i += kSwThreads) vv[i] = 0.0;
  __syncthreads();
  // b_0, read before the first cluster barrier: afterwards peers store y_0 over it
  for (int c = tid; c < B; c += kSwThreads) tv[c] = __ldcg(xs + c);
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) ticket[i] = -1;
    for (int i = 0; i < S; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cl_arrive();  // peers push into this CTA's shared memory only after it is initialised
  cl_wait();

  // --------------------------------------------------------- producer ---
  if (warp == kSwWarps) {
    long long pos = 0;
    for (int seg = 0; seg < nseg; ++seg) {
      int type, k;
      bool fwd;
      seg_info(seg, H, type, k, fwd);
      const int4* sch = L.sched + (rank * T_N + type) * kMaxSched;
      const int n = L.nsched[rank * T_N + type];
      const int4* tt = L.tiles[type & 1];
      const double* base = Fs + k * L.blk + ((type & 1) ? L.sub_off : 0);
      for (int p = 0; p < n; ++p, ++pos) {
        const int st = int(pos % S);
        if (pos >= S) mbar_wait(&empty[st], unsigned((pos / S) - 1) & 1u);
        if (lane == 0) {
          const int4 d = __ldg(tt + __ldg(&sch[p].x));
          const unsigned bytes = unsigned((d.z >> 16) * (d.z & 0xffff)) * 8u;
          ticket[st] = int(pos);  // stage st now belongs to position pos (its previous tile is released)
          mbar_expect_tx(&full[st], bytes);
          tma_bulk_load(stage + (size_t)st * kTileD, base + d.x, bytes, &full[st]);
        }
        __syncwarp();
      }
      // one cluster barrier closes every segment; arrive early, wait one late
      if (seg > 0) cl_wait();
      cl_arrive();
    }
    cl_wait();
    cl_arrive();  // final barrier
    cl_wait();
    return;
  }

  // -------------------------------------------------------- consumers ---
  long long pos = 0;
  double pre[kPre];
#pragma unroll
  for (int i = 0; i < kPre; ++i) pre[i] = 0.0;
  for (int seg = 0; seg < nseg; ++seg) {
    int type, k;
    bool fwd;
    seg_info(seg, H, type, k, fwd);
    const bool sub = type & 1, trans = type >= T_INVT;
    // prologue (vectors of the previous phase are complete: cluster barrier)
    bool sync = false;
    if (sub) {
#pragma unroll
      for (int i = 0; i < kPre; ++i) {
        const int c = tid + i * kSwWarps * 32;
        if (c < B) bv[c] = pre[i];
      }
      sync = true;
    } else if (fwd ? k < H - 1 : k > 0) {
      // prefetch the next phase's right-hand side: b_{k+1} (forward) / y_{k-1} (backward)
      const double* src = xs + (long long)(fwd ? k + 1 : k - 1) * B;
#pragma unroll
      for (int i = 0; i < kPre; ++i) {
        const int c = tid + i * kSwWarps * 32;
        pre[i] = c < B ? __ldcg(src + c) : 0.0;
      }
    }
    if (sync) consumers_sync();
    // forward INV: t -> y (tv -> vv), SUB: y -> t (vv -> tv); backward from
    // y_{H-1} in vv: INVT vv -> tv, SUBT tv -> vv.  A phase never writes the
    // vector it (or a slower peer) reads.
    const double* vec = (sub == fwd) ? vv : tv;
    double* dst = (sub == fwd) ? tv : vv;
    double* peer[CS];
#pragma unroll
    for (int q = 0; q < CS; ++q) peer[q] = CS > 1 ? cluster.map_shared_rank(dst, q) : dst;
    double* ys = xs + (long long)k * B;

    const int4* sch = L.sched + (rank * T_N + type) * kMaxSched;
    const int n = L.nsched[rank * T_N + type];
    const int4* tt = L.tiles[type & 1];
    double acc[kTile];
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll
    for (int r = 0; r < kTile; ++r) acc[r] = 0.0;
    for (int p = 0; p < n; ++p) {
      const int4 e = __ldg(sch + p);
      if ((e.y & 0xff) != warp) continue;
      const long long gp = pos + p;
      const int st = int(gp % S);
      const int4 d = __ldg(tt + e.x);
      const int I = d.y >> 16, J = d.y & 0xffff, h = d.z >> 16, wp = d.z & 0xffff;
      const bool act = 2 * lane < wp;
      const double* buf = stage + (size_t)st * kTileD;
      if (e.y & 0x100) {  // first tile of the output block
#pragma unroll
        for (int r = 0; r < kTile; ++r) acc[r] = 0.0;
        c0 = c1 = c2 = c3 = 0.0;
      }
      while (ticket[st] != int(gp)) {
      }
      mbar_wait(&full[st], unsigned(gp / S) & 1u);
      if (!trans) {  // row sums: acc[r] += T[r][2l..2l+1] . vec[64J + 2l..]
        if (act) {
          const double2 xv = reinterpret_cast<const double2*>(vec + J * kTile)[lane];
#pragma unroll
          for (int r = 0; r < kTile; ++r)
            if (r < h) {
              const double2 a = reinterpret_cast<const double2*>(buf + r * wp)[lane];
              acc[r] = fma(a.x, xv.x, fma(a.y, xv.y, acc[r]));
            }
        }
      } else if (act) {  // column sums: (c0, c1) += T[r][2l..2l+1] * vec[64I + r]
        const double* w = vec + I * kTile;
#pragma unroll 8
        for (int r = 0; r + 1 < h; r += 2) {
          const double2 a = reinterpret_cast<const double2*>(buf + r * wp)[lane];
          const double2 b = reinterpret_cast<const double2*>(buf + (r + 1) * wp)[lane];
          const double w0 = w[r], w1 = w[r + 1];
          c0 = fma(a.x, w0, c0);
          c1 = fma(a.y, w0, c1);
          c2 = fma(b.x, w1, c2);
          c3 = fma(b.y, w1, c3);
        }
        if (h & 1) {
          const double2 a = reinterpret_cast<const double2*>(buf + (h - 1) * wp)[lane];
          c0 = fma(a.x, w[h - 1], c0);
          c1 = fma(a.y, w[h - 1], c1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage
      if (e.y & 0x200) {  // last tile of the output block: finish it
        double v0, v1;
        int o;
        if (!trans) {
          butterfly64(acc, lane);
          v0 = acc[0], v1 = acc[1], o = I * kTile + 2 * lane;
        } else {
          v0 = c0 + c2, v1 = c1 + c3, o = J * kTile + 2 * lane;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int oo = o + u;
          if (oo < B) {
            const double val = sub ? bv[oo] - (u ? v1 : v0) : (u ? v1 : v0);
#pragma unroll
            for (int q = 0; q < CS; ++q) peer[q][oo] = val;
            if (!sub) ys[oo] = val;  // y_k (forward) / x_k (backward)
          }
        }
      }
    }
    pos += n;
    cl_arrive();  // results pushed: one cluster barrier (also a CTA barrier) ends the phase
    cl_wait();
  }
  cl_arrive();  // final barrier: no rank exits while peers may still touch its shared memory
  cl_wait();
}

// --------------------------------------------------------- compaction ---
struct TileTabs {
  const int4* tiles;  // INV tiles then SUB tiles
  int n_inv, n_all;
};

// Copy the dense column-major factor blocks (Linv_d: L_kk^-1, Lsub_d: L_{k+1,k})
// into the tile layout; record the largest magnitude of L_{k+1,k} outside the
// tiles (must be exactly zero).
__global__ void compact_factor_kernel(const double* __restrict__ Linv_d, const double* __restrict__ Lsub_d,
                                      double* __restrict__ F, TileTabs T, const int* __restrict__ jmin,
                                      long long sub_off, long long blk, int B, int H, int ns,
                                      unsigned long long* __restrict__ dropped) {
  const long long BB = (long long)B * B;
  const long long total = (long long)ns * H * blk;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long sk = e / blk;  // s * H + k
    const int k = int(sk % H);
    const long long w = e % blk;
    const bool sub = w >= sub_off;
    const long long ws = w - (sub ? sub_off : 0);
    int lo = sub ? T.n_inv : 0, hi = sub ? T.n_all : T.n_inv;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (T.tiles[mid].x <= ws) lo = mid; else hi = mid;
    }
    const int4 d = T.tiles[lo];
    const long long idx = ws - d.x;
    const int wp = d.z & 0xffff, h = d.z >> 16;
    double v = 0.0;
    if (idx < (long long)h * wp) {  // else: block-row alignment padding
      const int r = (d.y >> 16) * kTile + int(idx / wp), c = (d.y & 0xffff) * kTile + int(idx % wp);
      if (c < B) {
        if (!sub) v = c <= r ? Linv_d[sk * BB + (long long)c * B + r] : 0.0;
        else if (k < H - 1) v = Lsub_d[((sk / H) * (H - 1) + k) * BB + (long long)c * B + r];
      }
    }
    F[e] = v;
  }
  const long long tot2 = (long long)ns * (H - 1) * BB;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot2; e += (long long)gridDim.x * blockDim.x) {
    const long long m = e % BB;
    const int c = int(m / B), r = int(m % B);
    if (c < jmin[r / kTile] * kTile) {
      const double a = fabs(Lsub_d[e]);
      if (a != 0.0) atomicMax(dropped, (unsigned long long)__double_as_longlong(a));
    }
  }
}

void GpuSolver::build_sweep_layout() {
  const int H = G.H, nb = (B + kTile - 1) / kTile;
  if (B > kPre * kSwWarps * 32) throw Error(1, "interior block too large for the sweep kernel");
  // L_{k+1,k}: row r is zero left of c0(r) = (node(r) - 1)(P+1)
  std::vector<int> jmin(nb, nb);
  for (int r = 0; r < B; ++r) jmin[r / kTile] = std::min(jmin[r / kTile], std::max(0, r / NT - 1) * NT / kTile);
  auto hgt = [&](int I) { return std::min(kTile, B - I * kTile); };
  auto wpad = [&](int J) { return (std::min(kTile, B - J * kTile) + 1) & ~1; };
  std::vector<int4> tabs;
  std::vector<std::vector<int>> blocks[T_N];  // output block -> tile ids (into its table)
  for (auto& b : blocks) b.assign(nb, {});
  long long off = 0;
  for (int I = 0; I < nb; ++I)
    for (int J = 0; J <= I; ++J) {
      blocks[T_INV][I].push_back((int)tabs.size());
      blocks[T_INVT][J].push_back((int)tabs.size());
      tabs.push_back(make_int4((int)off, I << 16 | J, hgt(I) << 16 | wpad(J), 0));
      off += (long long)hgt(I) * wpad(J);
    }
  const int n_inv = (int)tabs.size();
  const long long sub_off = (off + 31) & ~31LL;  // 256-byte aligned
  off = 0;
  for (int I = 0; I < nb; ++I)
    for (int J = jmin[I]; J < nb; ++J) {
      const int id = (int)tabs.size() - n_inv;
      blocks[T_SUB][I].push_back(id);
      blocks[T_SUBT][J].push_back(id);
      tabs.push_back(make_int4((int)off, I << 16 | J, hgt(I) << 16 | wpad(J), 0));
      off += (long long)hgt(I) * wpad(J);
    }
  const long long blk = (sub_off + off + 31) & ~31LL;  // 256-byte aligned block rows
  if (blk >= (1LL << 31)) throw Error(1, "interior block too large for the sweep layout");
  // cluster size: about one wave of CTAs over the 148 SMs
  sweep_cs_ = NS >= 100 ? 1 : NS >= 48 ? 2 : NS >= 24 ? 4 : NS >= 12 ? 8 : 16;
  if (const char* e = std::getenv("SGW_SWEEP_CS")) {  // test hook: force a cluster size
    const int v = std::atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) sweep_cs_ = v;
  }
  if (sweep_cs_ == 16) {  // non-portable cluster size: only if 16-CTA clusters of this size are schedulable
    const size_t sm16 = (size_t)6 * kTileD * 8 + 16 * 8 + 4 * 8 + 3 * (size_t)nb * kTile * 8;
    const size_t smem = sm16 <= 227 * 1024 ? sm16 : (size_t)5 * kTileD * 8 + 16 * 8 + 4 * 8 + 3 * (size_t)nb * kTile * 8;
    int nclus = 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16), cfg.blockDim = dim3(kSwThreads), cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16, attr[0].val.clusterDim.y = 1, attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr, cfg.numAttrs = 1;
    if (cudaFuncSetAttribute((const void*)sweep_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
            cudaSuccess ||
        cudaFuncSetAttribute((const void*)sweep_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveClusters(&nclus, (const void*)sweep_kernel<16>, &cfg) != cudaSuccess || nclus < NS) {
      (void)cudaGetLastError();
      sweep_cs_ = 8;
    }
  }
  // schedules: output blocks -> (rank, warp) bins by longest-first greedy on
  // tile counts; each rank issues its warps' tiles interleaved
  const int CS = sweep_cs_, nbin = CS * kSwWarps;
  std::vector<int4> sched((size_t)CS * T_N * kMaxSched, make_int4(0, 0, 0, 0));
  std::vector<int> nsched((size_t)CS * T_N, 0);
  for (int t = 0; t < T_N; ++t) {
    std::vector<int> order(nb);
    for (int b = 0; b < nb; ++b) order[b] = b;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return blocks[t][a].size() > blocks[t][b].size(); });
    std::vector<long long> load(nbin, 0);
    std::vector<std::vector<int>> bins(nbin);
    for (int b : order) {
      if (blocks[t][b].empty()) continue;
      const int bi = int(std::min_element(load.begin(), load.end()) - load.begin());
      load[bi] += (long long)blocks[t][b].size();
      bins[bi].push_back(b);
    }
    for (int q = 0; q < CS; ++q) {
      std::vector<std::vector<int4>> perw(kSwWarps);
      for (int w = 0; w < kSwWarps; ++w)
        for (int b : bins[q * kSwWarps + w]) {
          const auto& tl = blocks[t][b];
          for (size_t i = 0; i < tl.size(); ++i)
            perw[w].push_back(make_int4(tl[i], w | int(i == 0) << 8 | int(i + 1 == tl.size()) << 9, b, 0));
        }
      int n = 0;
      for (size_t i = 0;; ++i) {
        bool any = false;
        for (int w = 0; w < kSwWarps; ++w)
          if (i < perw[w].size()) {
            if (n >= kMaxSched) throw Error(1, "sweep: schedule too long");
            sched[(size_t)(q * T_N + t) * kMaxSched + n++] = perw[w][i];
            any = true;
          }
        if (!any) break;
      }
      nsched[q * T_N + t] = n;
    }
  }
  std::vector<int> raw(tabs.size() * 4), sraw(sched.size() * 4);
  std::memcpy(raw.data(), tabs.data(), raw.size() * sizeof(int));
  std::memcpy(sraw.data(), sched.data(), sraw.size() * sizeof(int));
  sw_off.upload(raw);
  sw_cuts.upload(sraw);
  sw_ncut.upload(nsched);
  sw_cs.upload(jmin);
  SweepLayout L{};
  L.tiles[0] = reinterpret_cast<const int4*>(sw_off.p);
  L.tiles[1] = reinterpret_cast<const int4*>(sw_off.p) + n_inv;
  L.sched = reinterpret_cast<const int4*>(sw_cuts.p);
  L.nsched = sw_ncut.p;
  L.sub_off = sub_off, L.blk = blk, L.per_sub = (long long)H * blk;
  L.B = B, L.H = H, L.nb = nb, L.VL = nb * kTile;
  // ring depth: 6 x 32 KB stages when the shared memory (227 KB) allows (+1% at C2), else 5
  L.stages = (6LL * kTileD + 3LL * nb * kTile + 20) * 8 <= 227 * 1024 ? 6 : 5;
  if (const char* e = std::getenv("SGW_SWEEP_STAGES")) L.stages = std::max(2, std::min(8, std::atoi(e)));  // tuning hook
  L.n_inv = n_inv, L.n_all = (int)tabs.size();
  delete sweep_layout_;
  sweep_layout_ = new SweepLayout(L);
  Fcomp.alloc(size_t(NS) * L.per_sub);
  const size_t smem = sweep_smem_bytes();
  for (auto fn : {(const void*)sweep_kernel<1>, (const void*)sweep_kernel<2>, (const void*)sweep_kernel<4>,
                  (const void*)sweep_kernel<8>, (const void*)sweep_kernel<16>})
    SGW_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (sweep_cs_ == 16)
    SGW_CUDA(cudaFuncSetAttribute((const void*)sweep_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

// factor blocks of subdomains [b0, b0 + nb) (batch-local Linv / Lsub) -> tiles
void GpuSolver::compact_factor_batch(int b0, int nb) {
  const SweepLayout& L = *sweep_layout_;
  DBuf<unsigned long long> drop;
  drop.alloc(1);
  drop.zero(st_);
  TileTabs T{L.tiles[0], L.n_inv, L.n_all};
  compact_factor_kernel<<<8 * kNumSMs * 4, 256, 0, st_>>>(Linv.p, Lsub.p, Fcomp.p + (size_t)b0 * L.per_sub, T, sw_cs.p,
                                                           L.sub_off, L.blk, L.B, L.H, nb, drop.p);
  SGW_LAUNCHED();
  unsigned long long h = 0;
  SGW_CUDA(cudaMemcpyAsync(&h, drop.p, sizeof(h), cudaMemcpyDeviceToHost, st_));
  SGW_CUDA(cudaStreamSynchronize(st_));
  if (h != 0) {
    double v;
    std::memcpy(&v, &h, sizeof(v));
    throw Error(2, "interior factor: non-zero entry outside the block profile (" + std::to_string(v) + ")");
  }
  Linv.reset();
  Lsub.reset();
}

void destroy_sweep_layout(SweepLayout* p) { delete p; }

size_t GpuSolver::sweep_smem_bytes() const {
  const SweepLayout& L = *sweep_layout_;
  return (size_t)L.stages * kTileD * 8 + 16 * 8 + 4 * 8 + 3 * (size_t)L.VL * 8;
}

void GpuSolver::sweep(double* x) {
  const SweepLayout& L = *sweep_layout_;
  cudaEvent_t e0;
  KP.begin(K_SWEEP, st_, &e0);
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
  switch (sweep_cs_) {
    case 1: SGW_CUDA(cudaLaunchKernelEx(&cfg, sweep_kernel<1>, x, F, L)); break;
    case 2: SGW_CUDA(cudaLaunchKernelEx(&cfg, sweep_kernel<2>, x, F, L)); break;
    case 4: SGW_CUDA(cudaLaunchKernelEx(&cfg, sweep_kernel<4>, x, F, L)); break;
    case 8: SGW_CUDA(cudaLaunchKernelEx(&cfg, sweep_kernel<8>, x, F, L)); break;
    default: SGW_CUDA(cudaLaunchKernelEx(&cfg, sweep_kernel<16>, x, F, L)); break;
  }
  SGW_LAUNCHED();
  KP.end(st_);
}

// Algorithmic bytes of one forward + backward solve: every entry of the factor's
// profile read once per direction (L_kk^-1 lower triangle; L_{k+1,k} right of c0(r)).
double GpuSolver::bytes_sweep() const {
  const SweepLayout& L = *sweep_layout_;
  double inv = 0.5 * double(L.B) * (L.B + 1), sub = 0.0;
  for (int r = 0; r < L.B; ++r) sub += double(L.B - std::max(0, r / NT - 1) * NT);
  return 2.0 * 8.0 * double(NS) * (double(L.H) * inv + double(L.H - 1) * sub);
}

}  // namespace sgw
