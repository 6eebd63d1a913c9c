// Batched interior Dirichlet solve x <- A_II^-1 x for every subdomain
// (src/sg.cpp:317 and :350: SimplicialLLT::solve, restated block-wise).
//
// A_II = L L^T is block lower-bidiagonal over the H interior grid rows
// (blocks B = W (P+1), node-major / term-minor):
//   forward   y_k = L_kk^-1 (b_k - L_{k,k-1} y_{k-1})
//   backward  x_k = L_kk^-T (y_k - L_{k+1,k}^T x_{k+1})
// Every product is a row-major dot-product block stored compactly (row r holds
// columns cs(r) .. cs(r)+len(r)-1, cs even, len padded even -> 16-byte rows):
//   INV  = L_kk^-1          rows r: columns 0..r
//   SUB  = L_{k+1,k}        rows r: columns c0(r)..B-1, c0(r) = ((node(r)-1)(P+1))_even
//   INVT = L_kk^-T          rows c: columns c..B-1 (start rounded down to even)
//   SUBT = L_{k+1,k}^T      rows c: columns 0..rlen(c)-1, rlen(c) = #{r : c0(r) <= c}
// (entries outside the profile are exact zeros of the factor; checked at setup).
// The backward transposes double the capacity but not the traffic: each
// direction streams its own blocks once.
//
// Kernel: one thread-block cluster of CS CTAs per subdomain; rank q owns a
// contiguous row range of every block.  A producer warp streams the rank's
// rows through a ring of shared-memory stages with cp.async.bulk (TMA bulk
// copies completing on mbarriers) and keeps prefetching across block-row
// boundaries; 16 consumer warps compute one row each (128-bit shared loads,
// four accumulator chains, warp reduction) and push the result into every
// rank's copy of the vector through DSMEM; one split cluster barrier closes
// each block-row phase.
#include <cooperative_groups.h>

#include <cstdlib>
#include <cstring>

#include "solver.cuh"

namespace cg = cooperative_groups;

namespace sgw {

constexpr int kConsumerWarps = 16;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kSweepThreads = kConsumers + 32;  // + one TMA producer warp
constexpr int kMaxCuts = 1024;                  // chunk boundaries per (rank, block type)
enum { T_INV = 0, T_SUB = 1, T_INVT = 2, T_SUBT = 3, T_N = 4 };

struct SweepLayout {
  const int* off;   // [type][B+1] element offsets of the rows inside a block
  const int* cs;    // [type][B]   first column of each row
  const int* cuts;  // [(rank * T_N + type) * kMaxCuts + i]: chunk row boundaries
  const int* ncut;  // [rank * T_N + type]
  long long toff[T_N], blk, per_sub;  // type offset inside a block row, block-row stride, per subdomain
  int B, H, stages, stage_doubles;
  int lo[T_N][9];  // row split of each block type over the CS ranks
  int dbg;         // timing experiments only (SGW_SWEEP_DBG): 1 skip row math, 2 skip phase barriers
  int prefetch;    // chunks the L2 prefetch runs ahead of the smem ring
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
// Stage release: only orders this warp's shared-memory reads of the stage (already
// consumed into registers), so relaxed semantics suffice and the arrive does not
// wait for the warp's outstanding DSMEM pushes / global stores.
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// Streaming order: forward INV_0, SUB_0, INV_1, ..., INV_{H-1}; backward
// INVT_{H-1}, SUBT_{H-2}, INVT_{H-2}, ..., INVT_0.  SUB_k / SUBT_k hold
// L_{k+1,k} (block row k).
__device__ __forceinline__ void seg_info(int seg, int H, int& type, int& k, bool& fwd) {
  const int nf = 2 * H - 1;
  fwd = seg < nf;
  const int q = fwd ? seg : seg - nf;
  const int j = (q + 1) >> 1;
  const bool sub = q & 1;
  type = fwd ? (sub ? T_SUB : T_INV) : (sub ? T_SUBT : T_INVT);
  k = fwd ? (sub ? j - 1 : j) : H - 1 - j;
}

template <int CS, int S>
__global__ void __launch_bounds__(kSweepThreads) sweep_kernel(double* __restrict__ x, const double* __restrict__ F,
                                                              SweepLayout L) {
  extern __shared__ __align__(128) unsigned char smraw[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = CS > 1 ? (int)cluster.block_rank() : 0;
  const int s = blockIdx.x / CS;
  const int B = L.B, H = L.H, Bp = (B + 3) & ~1, STG = L.stage_doubles;
  double* stage = reinterpret_cast<double*>(smraw);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smraw + (size_t)S * STG * 8);
  unsigned long long* empty = full + 8;
  double* vv = reinterpret_cast<double*>(empty + 8);  // y_{k-1} (fwd) / x_{k+1} (bwd), zero padded
  double* tv = vv + Bp;                                 // intermediate t
  double* bv = tv + Bp;                                 // right-hand side block (b_{k+1} / y_k)
  int* soff = reinterpret_cast<int*>(bv + Bp);          // [T_N][Bp]
  int* scs = soff + T_N * Bp;                           // [T_N][Bp]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Fs = F + (long long)s * L.per_sub;
  double* xs = x + (long long)s * H * B;
  const int nseg = 2 * (2 * H - 1);

  for (int i = tid; i < 3 * Bp; i += kSweepThreads) vv[i] = 0.0;
  for (int t = 0; t < T_N; ++t)
    for (int i = tid; i <= B; i += kSweepThreads) {
      soff[t * Bp + i] = L.off[t * (B + 1) + i];
      if (i < B) scs[t * Bp + i] = L.cs[t * B + i];
    }
  if (tid == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], kConsumerWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cl_arrive();  // peers push into this CTA's shared memory only after it is initialised
  cl_wait();

  // --------------------------------------------------------- producer ---
  if (warp == kConsumerWarps) {
    int issued = 0;
    // L2 prefetch cursor running kPrefetch chunks ahead of the smem ring: under
    // full load HBM latency is ~3 us, so the ring refills from L2 instead
    int pseg = 0, pch = 0;
    auto prefetch_next = [&]() {
      while (pseg < nseg) {
        int t, kk;
        bool f;
        seg_info(pseg, H, t, kk, f);
        const int nct = L.ncut[rank * T_N + t];
        if (pch < nct) {
          const int* ct = L.cuts + (rank * T_N + t) * kMaxCuts;
          const int* of = soff + t * Bp;
          const int o0 = of[__ldg(ct + pch)], o1 = of[__ldg(ct + pch + 1)];
          const double* src = Fs + kk * L.blk + L.toff[t] + o0;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(unsigned(o1 - o0) * 8u)
                       : "memory");
          if (++pch == nct) pch = 0, ++pseg;
          return;
        }
        pch = 0;
        ++pseg;
      }
    };
    if (lane == 0)
      for (int i = 0; i < L.prefetch; ++i) prefetch_next();
    for (int seg = 0; seg < nseg; ++seg) {
      int type, k;
      bool fwd;
      seg_info(seg, H, type, k, fwd);
      const int* cut = L.cuts + (rank * T_N + type) * kMaxCuts;
      const int* off = soff + type * Bp;
      const double* base = Fs + k * L.blk + L.toff[type];
      const int nc = L.ncut[rank * T_N + type];
      for (int ch = 0; ch < nc; ++ch) {
        const int st = issued % S;
        if (issued >= S) mbar_wait(&empty[st], ((issued / S) - 1) & 1);
        if (lane == 0) {
          const int o0 = off[__ldg(cut + ch)], o1 = off[__ldg(cut + ch + 1)];
          const unsigned bytes = unsigned(o1 - o0) * 8u;
          mbar_expect_tx(&full[st], bytes);
          tma_bulk_load(stage + (size_t)st * STG, base + o0, bytes, &full[st]);
          if (L.prefetch) prefetch_next();
        }
        __syncwarp();
        ++issued;
      }
      // one cluster barrier closes every segment; arrive early, wait one late
      if (!(L.dbg & 2)) {
        if (seg > 0) cl_wait();
        cl_arrive();
      }
    }
    if (!(L.dbg & 2)) cl_wait();
    cl_arrive();  // final barrier
    cl_wait();
    return;
  }

  // -------------------------------------------------------- consumers ---
  int consumed = 0;
  for (int seg = 0; seg < nseg; ++seg) {
    int type, k;
    bool fwd;
    seg_info(seg, H, type, k, fwd);
    const bool sub = type == T_SUB || type == T_SUBT;
    const int* cut = L.cuts + (rank * T_N + type) * kMaxCuts;
    const int* off = soff + type * Bp;
    const int* cs = scs + type * Bp;
    const int nc = L.ncut[rank * T_N + type];
    // prologues
    bool synced = false;
    if (seg == 0) {  // b_0
      for (int c = tid; c < B; c += kConsumers) tv[c] = __ldcg(xs + c);
      synced = true;
    } else if (!fwd && k == H - 1 && !sub) {  // backward starts from y_{H-1}
      for (int c = tid; c < B; c += kConsumers) tv[c] = vv[c];
      synced = true;
    }
    if (sub) {  // right-hand side block: b_{k+1} (forward) or y_k (backward)
      const long long b0 = (long long)(fwd ? k + 1 : k) * B;
      for (int c = tid; c < B; c += kConsumers) bv[c] = __ldcg(xs + b0 + c);
      synced = true;
    }
    if (synced) consumers_sync();
    const double* vec = sub ? vv : tv;
    double* dst = sub ? tv : vv;

    for (int ch = 0; ch < nc; ++ch) {
      const int st = consumed % S;
      mbar_wait(&full[st], (consumed / S) & 1);
      const double* buf = stage + (size_t)st * STG;
      const int ra = __ldg(cut + ch), rb = __ldg(cut + ch + 1);
      const int o0 = off[ra];
      for (int r = ra + warp; r < ((L.dbg & 1) ? ra : rb); r += kConsumerWarps) {
        const double2* row = reinterpret_cast<const double2*>(buf + (off[r] - o0));
        const double2* v2 = reinterpret_cast<const double2*>(vec + cs[r]);
        const int n2 = (off[r + 1] - off[r]) >> 1;
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
        int q = lane;
        for (; q + 32 < n2; q += 64) {
          const double2 a = row[q], b = v2[q], c = row[q + 32], e = v2[q + 32];
          d0 += a.x * b.x;
          d1 += a.y * b.y;
          d2 += c.x * e.x;
          d3 += c.y * e.y;
        }
        if (q < n2) {
          const double2 a = row[q], b = v2[q];
          d0 += a.x * b.x;
          d1 += a.y * b.y;
        }
        const double d = warp_sum((d0 + d1) + (d2 + d3));
        // push the result row into every rank's copy (own + DSMEM peers)
        if (lane < CS) {
          const double val = sub ? bv[r] - d : d;
          (CS > 1 ? cluster.map_shared_rank(dst, lane) : dst)[r] = val;
          if (!sub && lane == 0) xs[(long long)k * B + r] = d;  // y_k or x_k
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage
      ++consumed;
    }
    if (!(L.dbg & 2)) {
      cl_arrive();  // results pushed: one cluster barrier (also a CTA barrier) ends the phase
      cl_wait();
    } else {
      consumers_sync();
    }
  }
  cl_arrive();  // final barrier: no rank exits while peers may still touch its shared memory
  cl_wait();
}

// --------------------------------------------------------- compaction ---
// Copy the dense column-major factor blocks (Linv_d: L_kk^-1, Lsub_d: L_{k+1,k})
// into the four compact row-major block types; record the largest magnitude
// met outside the SUB profile (must be exactly zero).
__global__ void compact_factor_kernel(const double* __restrict__ Linv_d, const double* __restrict__ Lsub_d,
                                      double* __restrict__ F, SweepLayout L, int ns,
                                      unsigned long long* __restrict__ dropped) {
  const int B = L.B, H = L.H;
  const long long BB = (long long)B * B;
  const long long total = (long long)ns * L.per_sub;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int s = int(e / L.per_sub);
    const long long o = e % L.per_sub;
    const int k = int(o / L.blk);
    const long long w = o % L.blk;
    int t = T_N - 1;
    while (w < L.toff[t]) --t;
    const long long ws = w - L.toff[t];
    const int* off = L.off + t * (B + 1);
    int lo = 0, hi = B;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (off[mid] <= ws) lo = mid; else hi = mid;
    }
    const int row = lo, col = L.cs[t * B + row] + int(ws - off[row]);
    double v = 0.0;
    const double* Li = Linv_d + ((long long)s * H + k) * BB;
    const double* Ls = Lsub_d + ((long long)s * (H - 1) + k) * BB;
    if (col < B) {
      if (t == T_INV && col <= row) v = Li[(long long)col * B + row];
      if (t == T_INVT && col >= row) v = Li[(long long)row * B + col];  // (L^-1)^T[row][col] = L^-1[col][row]
      if (k < H - 1) {
        if (t == T_SUB) v = Ls[(long long)col * B + row];
        if (t == T_SUBT) v = Ls[(long long)row * B + col];  // L^T[row][col] = L[col][row]
      }
    }
    F[e] = v;
  }
  const long long tot2 = (long long)ns * (H - 1) * BB;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot2; e += (long long)gridDim.x * blockDim.x) {
    const long long m = e % BB;
    const int c = int(m / B), r = int(m % B);
    if (c < L.cs[T_SUB * B + r]) {
      const double a = fabs(Lsub_d[e]);
      if (a != 0.0) atomicMax(dropped, (unsigned long long)__double_as_longlong(a));
    }
  }
}

// split rows [0, B) into CS contiguous ranges of ~equal element counts
static void split_rows(const std::vector<int>& off, int CS, int* lo) {
  const long long tot = off.back();
  int r = 0;
  lo[0] = 0;
  for (int q = 1; q < CS; ++q) {
    while (r < (int)off.size() - 1 && (long long)off[r] * CS < tot * q) ++r;
    lo[q] = r;
  }
  lo[CS] = (int)off.size() - 1;
}

// chunk boundaries: whole rows, at most `cap` doubles per chunk
static int cut_rows(const std::vector<int>& off, int lo, int hi, int cap, int* out) {
  int n = 0;
  out[0] = lo;
  int r = lo;
  while (r < hi) {
    int e = r + 1;
    while (e < hi && off[e + 1] - off[r] <= cap) ++e;
    out[++n] = e;
    r = e;
    if (n + 1 >= kMaxCuts) throw Error(1, "sweep: too many chunks");
  }
  return n;
}

void GpuSolver::build_compact_factor() {
  const int H = G.H;
  std::vector<int> c0(B), rlen(B, 0);
  for (int r = 0; r < B; ++r) c0[r] = std::max(0, (r / NT - 1) * NT) & ~1;
  for (int c = 0; c < B; ++c)
    for (int r = 0; r < B; ++r)
      if (c0[r] <= c) rlen[c] = r + 1;
  std::vector<int> off(T_N * (B + 1), 0), cs(T_N * B, 0);
  for (int t = 0; t < T_N; ++t)
    for (int r = 0; r < B; ++r) {
      int start = 0, len = 0;
      if (t == T_INV) start = 0, len = r + 1;
      if (t == T_SUB) start = c0[r], len = B - c0[r];
      if (t == T_INVT) start = r & ~1, len = B - (r & ~1);
      if (t == T_SUBT) start = 0, len = rlen[r];
      cs[t * B + r] = start;
      off[t * (B + 1) + r + 1] = off[t * (B + 1) + r] + ((len + 1) & ~1);
    }
  sw_off.upload(off);
  sw_cs.upload(cs);
  SweepLayout L{};
  L.off = sw_off.p, L.cs = sw_cs.p;
  long long acc = 0;
  for (int t = 0; t < T_N; ++t) {
    L.toff[t] = acc;
    acc += off[t * (B + 1) + B];
  }
  L.blk = acc;
  L.per_sub = (long long)H * L.blk;
  L.B = B, L.H = H;
  // cluster size: about one wave of CTAs over the 148 SMs; stage ring sized for
  // 1 CTA/SM (5 x 32 KB) or 2 CTAs/SM (3 x 16 KB) when there are more CTAs.
  sweep_cs_ = NS >= 100 ? 1 : NS >= 48 ? 2 : NS >= 24 ? 4 : 8;
  if (const char* e = std::getenv("SGW_SWEEP_CS")) {  // test hook: force a cluster size
    const int v = std::atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8) sweep_cs_ = v;
  }
  if (const char* e = std::getenv("SGW_SWEEP_DBG")) L.dbg = std::atoi(e);
  L.prefetch = 0;  // measured: L2 prefetch does not help at C2 (the consumers bound the rate)
  if (const char* e = std::getenv("SGW_SWEEP_PF")) L.prefetch = std::atoi(e);
  const bool two_per_sm = NS * sweep_cs_ > kNumSMs;
  L.stages = two_per_sm ? 3 : 5;
  L.stage_doubles = two_per_sm ? 2048 : 4096;
  if (B + 2 > L.stage_doubles) L.stage_doubles = (B + 2 + 15) & ~15, L.stages = 3;
  std::vector<int> cuts(size_t(sweep_cs_) * T_N * kMaxCuts, 0), ncut(size_t(sweep_cs_) * T_N, 0);
  for (int t = 0; t < T_N; ++t) {
    std::vector<int> ot(off.begin() + t * (B + 1), off.begin() + (t + 1) * (B + 1));
    split_rows(ot, sweep_cs_, L.lo[t]);
    for (int q = 0; q < sweep_cs_; ++q)
      ncut[q * T_N + t] = cut_rows(ot, L.lo[t][q], L.lo[t][q + 1], L.stage_doubles, &cuts[(q * T_N + t) * kMaxCuts]);
  }
  sw_cuts.upload(cuts);
  sw_ncut.upload(ncut);
  L.cuts = sw_cuts.p, L.ncut = sw_ncut.p;
  delete sweep_layout_;
  sweep_layout_ = new SweepLayout(L);
  Fcomp.alloc(size_t(NS) * L.per_sub);
  DBuf<unsigned long long> drop;
  drop.alloc(1);
  drop.zero(st_);
  compact_factor_kernel<<<8 * kNumSMs * 4, 256, 0, st_>>>(Linv.p, Lsub.p, Fcomp.p, L, NS, drop.p);
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
  const size_t smem = sweep_smem_bytes();
  for (auto fn : {(const void*)sweep_kernel<1, 5>, (const void*)sweep_kernel<2, 5>, (const void*)sweep_kernel<4, 5>,
                  (const void*)sweep_kernel<8, 5>, (const void*)sweep_kernel<1, 3>, (const void*)sweep_kernel<2, 3>,
                  (const void*)sweep_kernel<4, 3>, (const void*)sweep_kernel<8, 3>})
    SGW_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}

void destroy_sweep_layout(SweepLayout* p) { delete p; }

size_t GpuSolver::sweep_smem_bytes() const {
  const SweepLayout& L = *sweep_layout_;
  const int Bp = (L.B + 3) & ~1;
  return (size_t)L.stages * L.stage_doubles * 8 + 16 * 8 + 3 * (size_t)Bp * 8 + 2 * T_N * (size_t)Bp * 4;
}

void GpuSolver::sweep(double* x) {
  const SweepLayout& L = *sweep_layout_;
  cudaEvent_t e0;
  KP.begin(K_SWEEP, st_, &e0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(NS * sweep_cs_);
  cfg.blockDim = dim3(kSweepThreads);
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
  const bool s5 = L.stages == 5;
  switch (sweep_cs_) {
    case 1: SGW_CUDA(s5 ? cudaLaunchKernelEx(&cfg, sweep_kernel<1, 5>, x, F, L) : cudaLaunchKernelEx(&cfg, sweep_kernel<1, 3>, x, F, L)); break;
    case 2: SGW_CUDA(s5 ? cudaLaunchKernelEx(&cfg, sweep_kernel<2, 5>, x, F, L) : cudaLaunchKernelEx(&cfg, sweep_kernel<2, 3>, x, F, L)); break;
    case 4: SGW_CUDA(s5 ? cudaLaunchKernelEx(&cfg, sweep_kernel<4, 5>, x, F, L) : cudaLaunchKernelEx(&cfg, sweep_kernel<4, 3>, x, F, L)); break;
    default: SGW_CUDA(s5 ? cudaLaunchKernelEx(&cfg, sweep_kernel<8, 5>, x, F, L) : cudaLaunchKernelEx(&cfg, sweep_kernel<8, 3>, x, F, L)); break;
  }
  SGW_LAUNCHED();
  KP.end(st_);
}

double GpuSolver::bytes_sweep() const {
  // forward streams INV_0..H-1 + SUB_0..H-2, backward INVT + SUBT likewise
  const SweepLayout& L = *sweep_layout_;
  const double inv = double(L.toff[T_SUB] - L.toff[T_INV]) + double(L.blk - L.toff[T_SUBT]) * 0 +
                     double(L.toff[T_SUBT] - L.toff[T_INVT]);
  const double sub = double(L.toff[T_INVT] - L.toff[T_SUB]) + double(L.blk - L.toff[T_SUBT]);
  return 8.0 * double(NS) * (double(L.H) * inv + double(L.H - 1) * sub);
}

}  // namespace sgw
