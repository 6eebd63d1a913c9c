// Batched interior Dirichlet solve x <- A_II^-1 x for every subdomain
// (src/sg.cpp:317 and :350: SimplicialLLT::solve, restated block-wise).
//
// A_II = L L^T is block lower-bidiagonal over the H interior grid rows
// (blocks B = W (P+1), node-major / term-minor).  The factor is stored
// compactly, row-major, every row padded to an even length (16-byte aligned):
//   Linv_k = L_kk^-1        lower triangular: row r holds columns 0..r
//   Lsub_k = L_{k+1,k}      row r holds columns c0(r)..B-1 with
//                           c0(r) = max(0, (node(r)-1)(P+1)) rounded down to even
//                           (the dropped part is exactly zero; checked at setup)
// per subdomain: [Linv_0, Lsub_0, Linv_1, Lsub_1, ..., Linv_{H-1}].
//
// Kernel: one thread-block cluster of CS CTAs per subdomain; each rank owns a
// contiguous row range of every block.  The rank streams its rows through a
// ring of shared-memory stages filled by cp.async.bulk (TMA bulk copies)
// completing on mbarriers; the copy of the next chunk is issued as soon as a
// stage is consumed, so prefetch runs ahead across block-row boundaries while
// the cluster synchronises.  Forward rows are warp dot products; the backward
// (transposed) products accumulate column partials in registers from the
// same row-major rows and are reduced across the cluster through DSMEM.
#include <cooperative_groups.h>

#include <cstdlib>
#include <cstring>

#include "solver.cuh"

namespace cg = cooperative_groups;

namespace sgw {

constexpr int kConsumerWarps = 16;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kSweepThreads = kConsumers + 32;  // + one TMA producer warp
constexpr int kPairs = 2;  // column pairs per consumer thread in the transposed products (B <= 2048)
constexpr int kMaxCuts = 1024;  // chunk boundaries per (rank, block type)

struct SweepLayout {
  const long long* off_inv;  // B + 1 element offsets inside a Linv block
  const long long* off_sub;  // B + 1
  const int* c0;             // B
  const int* cuts;           // [(rank*2 + type) * kMaxCuts + i]: chunk row boundaries
  const int* ncut;           // [rank*2 + type]: chunks
  long long inv_len, sub_len, per_sub;
  int B, H, stages, stage_doubles;
  int inv_lo[9], sub_lo[9];  // row split of Linv / Lsub rows over the CS ranks
};

enum { T_INV = 0, T_SUB = 1 };

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
__device__ __forceinline__ void tma_bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// segment seg of the fixed streaming order: forward INV0, SUB0, INV1, SUB1, ...
// INV_{H-1}; backward INV_{H-1}, SUB_{H-2}, INV_{H-2}, ..., INV_0.
// Returns type and the factor block index (Lsub_k = L_{k+1,k} lives in block k).
__device__ __forceinline__ void seg_info(int seg, int H, int& type, int& k, bool& fwd) {
  const int nf = 2 * H - 1;
  fwd = seg < nf;
  const int q = fwd ? seg : seg - nf;
  if (q == 0) {
    type = T_INV;
    k = fwd ? 0 : H - 1;
    return;
  }
  const int j = (q + 1) >> 1;  // block-row step
  type = (q & 1) ? T_SUB : T_INV;
  if (fwd) k = (q & 1) ? j - 1 : j;   // SUB before INV_j is L_{j,j-1}
  else k = H - 1 - j;                 // SUB_k = L_{k+1,k}, then INV_k
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// split cluster barrier (release / acquire); legal for a cluster of one CTA
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait;" ::: "memory"); }
// barrier among the consumer warps only (the producer warp never joins)
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
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
  double* tv = vv + Bp;
  double* pA = tv + Bp;
  double* pB = pA + Bp;
  double* bv = pB + Bp;  // right-hand side block staged from global memory
  int* soff_inv = reinterpret_cast<int*>(bv + Bp);
  int* soff_sub = soff_inv + Bp;
  int* sc0 = soff_sub + Bp;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Fs = F + (long long)s * L.per_sub;
  double* xs = x + (long long)s * H * B;
  const long long blk = L.inv_len + L.sub_len;
  const int nseg = 2 * (2 * H - 1);
  const int* cut_t[2] = {L.cuts + (rank * 2 + T_INV) * kMaxCuts, L.cuts + (rank * 2 + T_SUB) * kMaxCuts};
  const int nct[2] = {L.ncut[rank * 2 + T_INV], L.ncut[rank * 2 + T_SUB]};

  for (int i = tid; i < 5 * Bp; i += kSweepThreads) vv[i] = 0.0;
  for (int i = tid; i <= B; i += kSweepThreads) {
    soff_inv[i] = int(L.off_inv[i]);
    soff_sub[i] = int(L.off_sub[i]);
    if (i < B) sc0[i] = L.c0[i];
  }
  if (tid == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&full[i], 1), mbar_init(&empty[i], kConsumerWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // --------------------------------------------------------- producer ---
  if (warp == kConsumerWarps) {
    int issued = 0;
    for (int seg = 0; seg < nseg; ++seg) {
      int type, k;
      bool fwd;
      seg_info(seg, H, type, k, fwd);
      const int* cut = cut_t[type];
      const int* off = type == T_SUB ? soff_sub : soff_inv;
      const double* base = Fs + k * blk + (type == T_SUB ? L.inv_len : 0);
      for (int ch = 0; ch < nct[type]; ++ch) {
        const int st = issued % S;
        if (issued >= S) mbar_wait(&empty[st], ((issued / S) - 1) & 1);
        if (lane == 0) {
          const int o0 = off[__ldg(cut + ch)], o1 = off[__ldg(cut + ch + 1)];
          const unsigned bytes = unsigned(o1 - o0) * 8u;
          mbar_expect_tx(&full[st], bytes);
          tma_bulk_load(stage + (size_t)st * STG, base + o0, bytes, &full[st]);
        }
        __syncwarp();
        ++issued;
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
  int consumed = 0;
  for (int seg = 0; seg < nseg; ++seg) {
    int type, k;
    bool fwd;
    seg_info(seg, H, type, k, fwd);
    const int* cut = cut_t[type];
    const int* off = type == T_SUB ? soff_sub : soff_inv;
    const int nc = nct[type];
    bool synced = false;
    if (type == T_INV && ((fwd && k == 0) || (!fwd && k == H - 1))) {
      if (fwd)
        for (int c = tid; c < B; c += kConsumers) tv[c] = __ldcg(xs + c);  // b_0
      else
        for (int c = tid; c < B; c += kConsumers) tv[c] = vv[c];           // y_{H-1}
      synced = true;
    }
    // right-hand side block of this segment: b_{k+1} rows (forward SUB) or y_k (backward SUB)
    if (type == T_SUB) {
      const long long b0 = (long long)(fwd ? k + 1 : k) * B;
      for (int c = tid; c < B; c += kConsumers) bv[c] = __ldcg(xs + b0 + c);
      synced = true;
    }
    if (synced) consumers_sync();
    double acc[kPairs][2];
#pragma unroll
    for (int j = 0; j < kPairs; ++j) acc[j][0] = acc[j][1] = 0.0;

    for (int ch = 0; ch < nc; ++ch) {
      const int st = consumed % S;
      mbar_wait(&full[st], (consumed / S) & 1);
      const double* buf = stage + (size_t)st * STG;
      const int ra = __ldg(cut + ch), rb = __ldg(cut + ch + 1);
      const int o0 = off[ra];
      if (fwd) {
        // warp per row: dot with the known vector
        const double* vec = type == T_SUB ? vv : tv;
        for (int r = ra + warp; r < rb; r += kConsumerWarps) {
          const int cf = type == T_SUB ? sc0[r] : 0;
          const double2* row = reinterpret_cast<const double2*>(buf + (off[r] - o0));
          const double2* v2 = reinterpret_cast<const double2*>(vec + cf);
          const int n2 = (off[r + 1] - off[r]) >> 1;
          double d = 0.0;
#pragma unroll 2
          for (int q = lane; q < n2; q += 32) {
            const double2 a = row[q], b = v2[q];
            d += a.x * b.x + a.y * b.y;
          }
          d = warp_sum(d);
          if (lane == 0) {
            if (type == T_SUB) {
              tv[r] = bv[r] - d;
            } else {
              vv[r] = d;
              xs[(long long)k * B + r] = d;
            }
          }
        }
      } else {
        // transposed product: column pairs owned by this thread
        for (int r = ra; r < rb; ++r) {
          const double* row = buf + (off[r] - o0);
          if (type == T_SUB) {
            const int c0 = sc0[r];
            const double w = vv[r];
#pragma unroll
            for (int j = 0; j < kPairs; ++j) {
              const int c = 2 * (tid + j * kConsumers);
              if (c < B && c >= c0) {
                const double2 a = *reinterpret_cast<const double2*>(row + (c - c0));
                acc[j][0] += a.x * w;
                acc[j][1] += a.y * w;
              }
            }
          } else {
            const double w = tv[r];
#pragma unroll
            for (int j = 0; j < kPairs; ++j) {
              const int c = 2 * (tid + j * kConsumers);
              if (c <= r) {
                const double2 a = *reinterpret_cast<const double2*>(row + c);
                acc[j][0] += a.x * w;
                acc[j][1] += a.y * w;
              }
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage
      ++consumed;
    }

    // segment epilogue: one cluster barrier, then exchange through DSMEM
    if (fwd) {
      cl_arrive();
      cl_wait();
      if (CS > 1) {
        const int* lo = type == T_SUB ? L.sub_lo : L.inv_lo;
        double* vec = type == T_SUB ? tv : vv;
        for (int q = 0; q < CS; ++q) {
          if (q == rank) continue;
          const double* rv = cluster.map_shared_rank(vec, q);
          for (int r = lo[q] + tid; r < lo[q + 1]; r += kConsumers) vec[r] = rv[r];
        }
      }
      consumers_sync();
    } else {
      double* part = type == T_SUB ? pA : pB;
#pragma unroll
      for (int j = 0; j < kPairs; ++j) {
        const int c = 2 * (tid + j * kConsumers);
        if (c < B) part[c] = acc[j][0], part[c + 1] = acc[j][1];
      }
      cl_arrive();
      cl_wait();
      const int per = (B + CS - 1) / CS, c_lo = rank * per, c_hi = min(B, c_lo + per);
      for (int c = tid; c < B; c += kConsumers) {
        double sum = 0.0;
        for (int q = 0; q < CS; ++q) sum += (CS > 1 ? cluster.map_shared_rank(part, q) : part)[c];
        if (type == T_SUB) {
          tv[c] = bv[c] - sum;  // y_k - L_{k+1,k}^T x_{k+1}
        } else {
          vv[c] = sum;  // x_k
          if (c >= c_lo && c < c_hi) xs[(long long)k * B + c] = sum;
        }
      }
      consumers_sync();
    }
  }
  cl_arrive();  // final barrier: no rank exits while its shared memory may be read
  cl_wait();
}

// Copy the dense column-major factor blocks into the compact row-major layout
// and record the largest magnitude among the dropped Lsub entries.
__global__ void compact_factor_kernel(const double* __restrict__ Linv_d, const double* __restrict__ Lsub_d,
                                      double* __restrict__ F, SweepLayout L, int ns,
                                      unsigned long long* __restrict__ dropped) {
  const int B = L.B, H = L.H;
  const long long BB = (long long)B * B;
  const long long total = (long long)ns * L.per_sub;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int s = int(e / L.per_sub);
    const long long o = e % L.per_sub;
    const long long blk = L.inv_len + L.sub_len;
    const int k = int(o / blk);
    const long long w = o % blk;
    double v = 0.0;
    if (w < L.inv_len) {  // Linv_k row-major
      int lo = 0, hi = B;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (L.off_inv[mid] <= w) lo = mid; else hi = mid;
      }
      const int r = lo, c = int(w - L.off_inv[r]);
      if (c <= r) v = Linv_d[((long long)s * H + k) * BB + (long long)c * B + r];
    } else {
      const long long ws = w - L.inv_len;
      int lo = 0, hi = B;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (L.off_sub[mid] <= ws) lo = mid; else hi = mid;
      }
      const int r = lo, c = L.c0[r] + int(ws - L.off_sub[r]);
      if (c < B && k < H - 1) v = Lsub_d[((long long)s * (H - 1) + k) * BB + (long long)c * B + r];
    }
    F[e] = v;
  }
  // dropped entries of Lsub (columns < c0(r)) must be exact zeros
  const long long tot2 = (long long)ns * (H - 1) * BB;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot2; e += (long long)gridDim.x * blockDim.x) {
    const long long m = e % BB;
    const int c = int(m / B), r = int(m % B);
    if (c < L.c0[r]) {
      const double a = fabs(Lsub_d[e]);
      if (a != 0.0) atomicMax(dropped, (unsigned long long)__double_as_longlong(a));
    }
  }
}

// split rows [0, B) into CS contiguous ranges of ~equal element counts
static void split_rows(const std::vector<long long>& off, int CS, int* lo) {
  const long long tot = off.back();
  int r = 0;
  lo[0] = 0;
  for (int q = 1; q < CS; ++q) {
    while (r < (int)off.size() - 1 && off[r] * CS < tot * q) ++r;
    lo[q] = r;
  }
  lo[CS] = (int)off.size() - 1;
}

// chunk boundaries: whole rows, at most `cap` doubles per chunk
static int cut_rows(const std::vector<long long>& off, int lo, int hi, int cap, int* out) {
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
  std::vector<long long> oi(B + 1, 0), os(B + 1, 0);
  std::vector<int> c0(B);
  for (int r = 0; r < B; ++r) {
    const int node = r / NT;
    c0[r] = std::max(0, (node - 1) * NT) & ~1;  // even start: 16-byte aligned column pairs
    oi[r + 1] = oi[r] + ((r + 1 + 1) & ~1);
    os[r + 1] = os[r] + ((B - c0[r] + 1) & ~1);
  }
  sw_off_inv.upload(oi);
  sw_off_sub.upload(os);
  sw_c0.upload(c0);
  SweepLayout L{};
  L.off_inv = sw_off_inv.p, L.off_sub = sw_off_sub.p, L.c0 = sw_c0.p;
  L.inv_len = oi[B], L.sub_len = os[B];
  L.per_sub = H * L.inv_len + (H - 1) * L.sub_len;
  L.B = B, L.H = H;
  // cluster size: about one wave of CTAs over the 148 SMs; stage ring sized for
  // 1 CTA/SM (5 x 32 KB) or 2 CTAs/SM (4 x 16 KB) when there are more CTAs.
  sweep_cs_ = NS >= 100 ? 1 : NS >= 48 ? 2 : NS >= 24 ? 4 : 8;
  if (const char* e = std::getenv("SGW_SWEEP_CS")) {  // test hook: force a cluster size
    const int v = std::atoi(e);
    if (v == 1 || v == 2 || v == 4 || v == 8) sweep_cs_ = v;
  }
  const bool two_per_sm = NS * sweep_cs_ > kNumSMs;
  L.stages = two_per_sm ? 3 : 5;
  L.stage_doubles = two_per_sm ? 2048 : 4096;
  if (B + 2 > L.stage_doubles) L.stage_doubles = (B + 2 + 15) & ~15, L.stages = 3;
  split_rows(oi, sweep_cs_, L.inv_lo);
  split_rows(os, sweep_cs_, L.sub_lo);
  std::vector<int> cuts(size_t(sweep_cs_) * 2 * kMaxCuts, 0), ncut(size_t(sweep_cs_) * 2, 0);
  for (int q = 0; q < sweep_cs_; ++q) {
    ncut[q * 2 + 0] = cut_rows(oi, L.inv_lo[q], L.inv_lo[q + 1], L.stage_doubles, &cuts[(q * 2 + 0) * kMaxCuts]);
    ncut[q * 2 + 1] = cut_rows(os, L.sub_lo[q], L.sub_lo[q + 1], L.stage_doubles, &cuts[(q * 2 + 1) * kMaxCuts]);
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
  return (size_t)L.stages * L.stage_doubles * 8 + 16 * 8 + 5 * (size_t)Bp * 8 + 3 * (size_t)Bp * 4;
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
  // forward + backward stream the compact factor once each
  const SweepLayout& L = *sweep_layout_;
  return 2.0 * 8.0 * double(NS) * double(L.per_sub);
}

}  // namespace sgw
