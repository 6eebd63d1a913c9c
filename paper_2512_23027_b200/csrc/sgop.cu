// Fused stochastic-Galerkin operator apply (src/sg.cpp:425-447):
//   y_k = alpha sum_e M^e x_k  +  beta sum_{(i,j)} c_ijk sum_e K_i^e x_j  (+ gamma sum_e M^e x2_k)
// on a batch of structured node grids, e over the P1 stencil (5 points for K,
// 7 for M).  The kernel is generated and compiled at setup (NVRTC, sm_100a)
// for the solver's triple-product tensor, so every (i, j) pair and every
// c_ijk becomes straight-line code with the PCE terms in named registers:
//
//   * CTA = a tile of 32 x R nodes of one grid; G threads per node split the
//     input terms j (balanced by pair count).  A thread keeps the 5-point
//     neighbourhoods of its j's in registers for the whole tile and
//     accumulates all (P+1) outputs.
//   * K_i stencils (3 stored components per node) stream through a ring of
//     shared-memory stages, a chunk of input terms i per stage, with
//     cp.async (16-byte, zero-filled outside the grid); x tiles and M are
//     staged per tile (double-buffered across tiles).  Per node and i: 5
//     shared loads, then 5 FMAs per (i, j) pair and 1 per c_ijk.
//   * The G partial outputs of a node are summed in shared memory in fixed
//     group order (bitwise reproducible); coalesced stores.
// K / M live in a padded layout [item][i][c][row][pitch] (pitch even, zero
// padding); x / y in the caller's layout (any pitch, term and item strides).
#include <nvrtc.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>

#include "solver.cuh"

namespace sgw {

namespace {
const char* kDeviceTemplate = R"CUDA(
typedef long long ll;
struct SgOpArgs {
  const double* K; const double* M;  // tiled stencils (sgop_tile_stencils)
  const double* xt;                  // tiled input (sgop_pack_x): [tile][NT][R+2][34]
  const double* x; const double* x2; double* y;
  ll xterm, xitem, yterm, yitem;
  int W, H, xpitch, ypitch, tiles_x, tiles_y, items;
  double alpha, beta, gamma;
  const double* Mg;                  // mass stencils in grid layout [item][4][H][W]
};
#define XW 34
#define RUP16(v) (((v) + 15) / 16 * 16)
#define XBUF RUP16(NT * (R + 2) * XW)
/* per tile and input term: diag [R][32], E [R][33] (from column -1), N [R+1][32] (from row -1) */
#define KOE (32 * R)
#define KON (32 * R + 33 * R)
#define KPI ((97 * R + 32 + 1) / 2 * 2)
/* M per tile: diag, E, N as K, then NE [R+1][33] (from row -1, column -1) */
#define MON (32 * R + 33 * R)
#define MONE (97 * R + 32)
#define MPI ((130 * R + 65 + 1) / 2 * 2)
#define MBUF RUP16(MPI)
#define KSTG RUP16(IC * KPI)
#define NODES (32 * R)
#define NC (R * G)                 /* consumer warps; PROD: warp NC feeds the pipeline, else warp 0 */
#define NTHR (32 * (NC + PROD))

extern __shared__ __align__(1024) double sm[];
#if XG
/* x and M come from global memory (L2-resident): the ring holds only K */
#define KS (sm)
#define REDSEP (sm + S * KSTG)
#else
#define XS (sm)
#define MS (sm + 2 * XBUF)
#define KS (sm + 2 * XBUF + 2 * MBUF)
#define REDSEP (sm + 2 * XBUF + 2 * MBUF + S * KSTG)
#endif
#define BARS ((unsigned long long*)(REDSEP + (RED_ALIAS ? 0 : (G - 1) * NT * NODES)))
#define KFULL(i) (BARS + (i))
#define KEMPTY(i) (BARS + S + (i))
#define XFULL(i) (BARS + 2 * S + (i))
#define XEMPTY(i) (BARS + 2 * S + 2 + (i))
#define KCNT ((int*)(BARS + 2 * S + 4))  /* LA: per-stage release counters */
__constant__ double gcoef[NCOEF];

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp8(double* s, const double* g, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" :: "r"(su(s)), "l"(g), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void bulk(double* s, const double* g, unsigned bytes, unsigned long long* bar) {
#if EF
  /* stencils stream once per apply: evict-first keeps x and M resident in L2 */
  asm volatile("{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
               " cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}"
               :: "r"(su(s)), "l"(g), "r"(bytes), "r"(su(bar)) : "memory");
#else
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(su(s)), "l"(g), "r"(bytes), "r"(su(bar)) : "memory");
#endif
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(su(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(su(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {  // release: prior reads done
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
               :: "r"(su(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" :: "n"(NC * 32) : "memory"); }

__device__ __forceinline__ void tile_coords(const SgOpArgs& A, int t, int& tx, int& ty, int& it) {
  const int tile = blockIdx.x + t * gridDim.x;
  tx = tile % A.tiles_x, ty = (tile / A.tiles_x) % A.tiles_y, it = tile / (A.tiles_x * A.tiles_y);
}

// x tile and M block of tile t into buffer t & 1 (two bulk copies, lane 0).
__device__ __forceinline__ void load_xm(const SgOpArgs& A, int t, int lane) {
  if (XG || lane != 0) return;
  if (t >= 2) mbar_wait(XEMPTY(t & 1), (unsigned)((t >> 1) - 1) & 1u);
  const ll tile = blockIdx.x + t * gridDim.x;
  mbar_expect_tx(XFULL(t & 1), (unsigned)((XBUF + MPI) * 8));
#if !XG
  bulk(XS + (t & 1) * XBUF, A.xt + tile * XBUF, XBUF * 8, XFULL(t & 1));
  bulk(MS + (t & 1) * MBUF, A.M + tile * MPI, MPI * 8, XFULL(t & 1));
#endif
}

// K chunk q (stage q % S) of this CTA: IC input terms of its tile q / NCHUNK.
// K is stored tile by tile ([tile][i][KPI]): one contiguous bulk copy, issued
// by lane 0 of warp 0 once every warp has released the stage's previous use.
__device__ __forceinline__ const double* k_chunk(const SgOpArgs& A, int q, unsigned& bytes) {
  const int t = q / NCHUNK, ch = q % NCHUNK;
  bytes = (unsigned)(min(IC, NIN - ch * IC) * KPI * 8);
  return A.K + ((ll)(blockIdx.x + t * gridDim.x) * NIN + (ll)ch * IC) * KPI;
}
__device__ __forceinline__ void issue_k(const SgOpArgs& A, int q, int nst, int lane) {
  if (lane != 0) return;
  if (q + PF < nst) {  // L2 prefetch PF chunks beyond the ring: HBM latency under load is ~4 us
    unsigned b;
    const double* src = k_chunk(A, q + PF, b);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(src), "r"(b) : "memory");
  }
  if (q >= nst) return;
  if (q >= S) mbar_wait(KEMPTY(q % S), (unsigned)((q / S) - 1) & 1u);
  unsigned bytes;
  const double* src = k_chunk(A, q, bytes);
  mbar_expect_tx(KFULL(q % S), bytes);
  bulk(KS + (q % S) * KSTG, src, bytes, KFULL(q % S));
}

// LA: issue chunk q into its (released) stage, no wait
__device__ __forceinline__ void issue_k_now(const SgOpArgs& A, int q, int nst) {
  if (q >= nst) return;
  unsigned bytes;
  const double* src = k_chunk(A, q, bytes);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(KFULL(q % S), bytes);
  bulk(KS + (q % S) * KSTG, src, bytes, KFULL(q % S));
}

// shared-memory reads of the current tile: x (center at [ly+1][lane+1]);
// K of input term ii: own diag / E / N, west neighbour's E, south neighbour's N;
// M likewise plus own NE and the south-west neighbour's NE
#define XV(j, dy, dx) xb[((j) * (R + 2) + ly + 1 + (dy)) * XW + lane + 1 + (dx)]
#define K_D(ii) kb[(ii) * KPI + ly * 32 + lane]
#define K_E(ii) kb[(ii) * KPI + KOE + ly * 33 + lane + 1]
#define K_W(ii) kb[(ii) * KPI + KOE + ly * 33 + lane]
#define K_N(ii) kb[(ii) * KPI + KON + (ly + 1) * 32 + lane]
#define K_S(ii) kb[(ii) * KPI + KON + ly * 32 + lane]
#if PROD
// the producer warp runs the ring ahead; consumers only wait for their chunk
#define STAGE_IN(ch)                                                   \
  mbar_wait(KFULL(s % S), (unsigned)(s / S) & 1u);                     \
  kb = KS + (s % S) * KSTG;
#elif LA
#define STAGE_IN(ch)                                                   \
  if (warp == 0 && (ch) == NCHUNK / 2 && t + 1 < mytiles) {            \
    load_xm(A, t + 1, lane);                                           \
    __syncwarp();                                                      \
  }                                                                    \
  mbar_wait(KFULL(s % S), (unsigned)(s / S) & 1u);                     \
  kb = KS + (s % S) * KSTG;
#else
// warp 0 feeds the ring S - 2 chunks ahead (and the next tile's x / M at
// mid-tile), then every warp waits for its chunk
#define STAGE_IN(ch)                                                   \
  if (warp == 0) {                                                     \
    issue_k(A, s + AHEAD, nst, lane);                                  \
    if ((ch) == NCHUNK / 2 && t + 1 < mytiles) load_xm(A, t + 1, lane); \
    __syncwarp();                                                      \
  }                                                                    \
  mbar_wait(KFULL(s % S), (unsigned)(s / S) & 1u);                     \
  kb = KS + (s % S) * KSTG;
#endif
#if LA
// the last warp to release a stage refills it at once (S chunks in flight)
#define STAGE_OUT()                                                    \
  __syncwarp();                                                        \
  if (lane == 0) {                                                     \
    __threadfence_block();                                             \
    if (atomicAdd(KCNT + s % S, 1) == NC - 1) {                        \
      KCNT[s % S] = 0;                                                 \
      issue_k_now(A, s + S, nst);                                      \
    }                                                                  \
  }                                                                    \
  ++s;
#else
#define STAGE_OUT()                                                    \
  __syncwarp();                                                        \
  if (lane == 0) mbar_arrive(KEMPTY(s % S));                           \
  ++s;
#endif

// producer warp: per tile its x / M buffer, then the tile's K chunks, paced by
// the consumers' releases
__device__ __forceinline__ void producer(const SgOpArgs& A, int mytiles, int nst, int lane) {
  int q = 0;
  for (int t = 0; t < mytiles; ++t) {
    load_xm(A, t, lane);
    for (int ch = 0; ch < NCHUNK; ++ch, ++q) issue_k(A, q, nst, lane);
  }
}

@GROUPS@

extern "C" __global__ void __launch_bounds__(NTHR, CPS) sgop_kernel(const SgOpArgs A) {
  const int ntiles = A.tiles_x * A.tiles_y * A.items;
  if ((int)blockIdx.x >= ntiles) return;
  const int mytiles = (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nst = mytiles * NCHUNK;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(KFULL(i), 1), mbar_init(KEMPTY(i), NC), KCNT[i] = 0;
    for (int i = 0; i < 2; ++i) mbar_init(XFULL(i), 1), mbar_init(XEMPTY(i), NC);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
#if PROD
  if (warp == NC) {
    producer(A, mytiles, nst, lane);
    return;
  }
#elif LA
  if (threadIdx.x == 0)
    for (int q = 0; q < S; ++q) issue_k_now(A, q, nst);
  if (warp == 0) {
    load_xm(A, 0, lane);
    __syncwarp();
  }
#else
  if (warp == 0) {
    for (int q = 0; q < AHEAD; ++q) issue_k(A, q, nst, lane);
    load_xm(A, 0, lane);
    __syncwarp();
  }
#endif
  const int ly = warp / G, gq = warp % G;
  @DISPATCH@
}
)CUDA";

std::string dlit(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  std::string s(b);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}
}  // namespace

struct SgOpJit {
  int NT = 0, NIN = 0, R = 4, G = 2, IC = 4, S = 6, NCHUNK = 0, regs = 255, prod = 0, la = 0;
  int cps = 1;  // CTAs per SM (shared memory and registers split between them)
  bool red_alias = true;  // partial sums reuse the tile's x buffer (after the mass step)
  bool jouter = false;    // k-resident code shape (see sgop_source)
  bool xg = true;         // x and M read from global memory (no packed x tiles, K-only ring)
  size_t smem = 0;
  std::vector<double> coef;  // c_ijk in generated order (__constant__ gcoef)
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  ~SgOpJit() {
    if (lib) cudaLibraryUnload(lib);
  }
};

// shared memory: x tiles (2), M tiles (2), K ring (S stages), partial-sum buffer
static long long sgop_smem_doubles(const SgOpJit& J) {
  const long long xw = 34;
  auto up = [](long long v) { return (v + 15) / 16 * 16; };
  const long long kpi = (97LL * J.R + 33) / 2 * 2, mpi = (130LL * J.R + 66) / 2 * 2;
  if (J.xg) return J.S * up((long long)J.IC * kpi) + (long long)(J.G - 1) * J.NT * 32 * J.R + 3 * J.S + 4;
  return 2 * up(J.NT * (J.R + 2) * xw) + 2 * up(mpi) + J.S * up((long long)J.IC * kpi) +
         (J.red_alias ? 0 : (long long)(J.G - 1) * J.NT * 32 * J.R) + 3 * J.S + 4;  // + barriers, counters
}

// CUDA source of the operator specialised for (NT, NIN, T); fills J's shape.
std::string sgop_source(int NT, int NIN, const TensorHost& T, SgOpJit* J) {
  J->NT = NT, J->NIN = NIN;
  if (const char* e = std::getenv("SGW_SGOP_CPS")) J->cps = std::max(1, std::min(4, std::atoi(e)));  // tuning hook
  // <= 7 input terms (35 neighbourhood values) per thread; threads per CTA
  // bounded by the register file (estimate: x and y live values + 40) and
  // the shared memory by the tile height R
  // <= 10 input terms per thread; the tile height R from the register file
  // (estimate: x and y live values + 60); then as many K stages as the
  // shared memory holds (bytes in flight set the achievable HBM rate)
  // Threads of a node: GJ groups of input terms j (registers: 5 neighbourhood
  // values per j) times GI interleaved groups of input terms i (shorter code
  // per thread; with G = 4 every SM sub-partition runs a single code stream).
  // Two code shapes.  "x-resident" (default): a thread keeps the 5-point
  // neighbourhoods of its j's in registers for the whole tile and streams
  // K_i.  "k-resident" (SGW_SGOP_MODE=jout): threads keep the stencils of a
  // chunk of IC input terms in registers and read each x_j neighbourhood
  // once per chunk from shared memory (fewer registers, more shared-memory
  // traffic; measured 12% slower at C2).
  J->jouter = false;
  if (const char* e = std::getenv("SGW_SGOP_MODE")) J->jouter = std::string(e) == "jout";  // tuning hook
  int GJ = J->jouter ? 2 : (NT + 9) / 10, GI = 1;
  if (const char* e = std::getenv("SGW_SGOP_G")) GJ = std::max(1, std::atoi(e));   // tuning hooks
  if (const char* e = std::getenv("SGW_SGOP_GI")) GI = std::max(1, std::atoi(e));
  if (J->jouter) GI = 1;
  if (GJ > 6) return std::string();  // larger PCE bases: the generic kernel (step.cu)
  J->G = GJ * GI;
  J->IC = J->jouter ? 4 : NIN >= 64 ? 16 : NIN >= 48 ? 12 : NIN >= 24 ? 4 : 2;  // measured at C2 (L2 flushed): 16 best
  if (const char* e = std::getenv("SGW_SGOP_IC")) J->IC = std::max(1, std::atoi(e));  // tuning hook
  const int jg = (NT + GJ - 1) / GJ;
  const int est = J->jouter ? 2 * (5 * J->IC + NT + 5) + 60 : 2 * (5 * jg + NT) + 80;
  J->NCHUNK = (NIN + J->IC - 1) / J->IC;
  J->R = std::max(1, std::min(16, 65536 / J->cps / est / (32 * J->G)));
  if (const char* e = std::getenv("SGW_SGOP_PROD")) J->prod = std::atoi(e) != 0;  // tuning hook: producer warp
  if (const char* e = std::getenv("SGW_SGOP_LA")) J->la = std::atoi(e) != 0;      // tuning hook: last-arriver refill
  if (J->prod) J->la = 0;
  if (const char* e = std::getenv("SGW_SGOP_R")) J->R = std::max(1, std::atoi(e));  // tuning hook
  const long long budget = 220 * 1024 / 8 / J->cps;
  if (const char* e = std::getenv("SGW_SGOP_XG")) J->xg = std::atoi(e) != 0;  // tuning hook
  if (J->jouter) J->xg = false;
  for (;; --J->R) {
    J->red_alias = !J->xg && (long long)(J->G - 1) * NT * 32 * J->R <= (long long)NT * (J->R + 2) * 34;
    J->S = 3;
    if (sgop_smem_doubles(*J) <= budget || J->R == 1) break;
  }
  while (J->S < 12 && J->S <= J->NCHUNK) {
    ++J->S;
    if (sgop_smem_doubles(*J) > budget) {
      --J->S;
      break;
    }
  }
  if (const char* e = std::getenv("SGW_SGOP_S")) J->S = std::max(3, std::atoi(e));  // tuning hook
  // registers are split per SM sub-partition: the warp count per partition sets the cap
  J->regs = std::min(255, 16384 / (32 * J->cps * ((J->R * J->G + J->prod + 3) / 4)) & ~7);
  const int R = J->R, G = J->G, IC = J->IC;
  // full (i, j) -> [(k, c)] expansion of the j <= k tensor (pce.hpp:24-40)
  std::map<std::pair<int, int>, std::vector<std::pair<int, double>>> pairs;
  for (size_t e = 0; e < T.v.size(); ++e) {
    pairs[{T.i[e], T.j[e]}].push_back({T.k[e], T.v[e]});
    if (T.j[e] != T.k[e]) pairs[{T.i[e], T.k[e]}].push_back({T.j[e], T.v[e]});
  }
  // j groups balanced by work (5 FMAs per pair + 1 per coefficient)
  std::vector<long long> wj(NT, 0);
  for (auto& p : pairs) wj[p.first.second] += 5 + (long long)p.second.size();
  std::vector<int> order(NT), grp(NT, 0);
  for (int j = 0; j < NT; ++j) order[j] = j;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return wj[a] > wj[b]; });
  std::vector<long long> load(GJ, 0);
  for (int j : order) {
    const int g = int(std::min_element(load.begin(), load.end()) - load.begin());
    grp[j] = g;  // j group; the owner of output k = j is group grp[k] (i group 0)
    load[g] += wj[j] + 7;
  }
  // timing experiment only (SGW_SGOP_DBG=1): stream and synchronise, skip the stencil math
  const bool dbg_nomath = std::getenv("SGW_SGOP_DBG") && std::atoi(std::getenv("SGW_SGOP_DBG")) == 1;
  // per pair: one 5-FMA chain (fewest issue slots) or two chains plus an add
  // interleaving: NI input terms per block, NIL pair chains in flight
  int NI = 2, NIL = 4;
  bool lit = true;  // c_ijk as literals in the code (immediates when short) instead of constant-bank loads
  if (const char* e = std::getenv("SGW_SGOP_LIT")) lit = std::atoi(e) != 0;  // tuning hook
  if (const char* e = std::getenv("SGW_SGOP_NI")) NI = std::max(1, std::atoi(e));    // tuning hooks
  if (const char* e = std::getenv("SGW_SGOP_NIL")) NIL = std::max(1, std::atoi(e));
  // generated per-group tile loops
  std::string groups, dispatch = "switch (gq) {\n";
  for (int g = 0; g < G; ++g) {
    const int jgrp = g % GJ, igrp = g / GJ;
    const bool owner = igrp == 0;  // owns the outputs k of its j group
    std::vector<int> js;
    for (int j = 0; j < NT; ++j)
      if (grp[j] == jgrp) js.push_back(j);
    std::string c;
    c += "__device__ __forceinline__ void group" + std::to_string(g) +
         "(const SgOpArgs& A, int ly, int lane, int warp, int mytiles, int nst) {\n";
    c += "  int s = 0;\n  for (int t = 0; t < mytiles; ++t) {\n";
    c += "    const int tile = blockIdx.x + t * gridDim.x;\n";
    c += "    const int tx = tile % A.tiles_x, ty = (tile / A.tiles_x) % A.tiles_y, it = tile / (A.tiles_x * A.tiles_y);\n";
    if (J->xg) {
      c += "    const int gx = tx * 32 + lane, gy = ty * R + ly;\n";
      c += "    const bool valid = gx < A.W && gy < A.H;\n";
      c += "    const bool hw = valid && gx > 0, he = valid && gx + 1 < A.W, hs = valid && gy > 0, hn = valid && gy + 1 < A.H;\n";
      c += "    const double* xg = A.x + it * A.xitem + (ll)(valid ? gy : 0) * A.xpitch + (valid ? gx : 0);\n";
      c += "#define XGV(j, dy, dx, ok) ((ok) ? __ldg(xg + (j) * A.xterm + (dy) * A.xpitch + (dx)) : 0.0)\n";
    } else {
      c += "    double* xb = XS + (t & 1) * XBUF;\n    const double* mb = MS + (t & 1) * MBUF;\n";
    }
    c += "    const double* kb;\n    (void)tx, (void)ty;\n";
    for (int ch = 0; ch < J->NCHUNK; ++ch) {
      if (ch == 0 && J->xg && !J->jouter)  // neighbourhoods from global memory before the first wait
        for (int j : js) {
          const std::string J0 = std::to_string(j);
          c += "    const double x" + J0 + "c = XGV(" + J0 + ", 0, 0, valid), x" + J0 + "e = XGV(" + J0 +
               ", 0, 1, he), x" + J0 + "w = XGV(" + J0 + ", 0, -1, hw), x" + J0 + "n = XGV(" + J0 +
               ", 1, 0, hn), x" + J0 + "s = XGV(" + J0 + ", -1, 0, hs);\n";
        }
      if (ch == 0 && !J->xg)  // x / M of this tile
        c += "    mbar_wait(XFULL(t & 1), (unsigned)(t >> 1) & 1u);\n";
      c += "    STAGE_IN(" + std::to_string(ch) + ");\n";
      if (ch == 0 && !J->jouter && !J->xg) {
        for (int j : js) {
          const std::string J0 = std::to_string(j);
          c += "    const double x" + J0 + "c = XV(" + J0 + ", 0, 0), x" + J0 + "e = XV(" + J0 + ", 0, 1), x" + J0 +
               "w = XV(" + J0 + ", 0, -1), x" + J0 + "n = XV(" + J0 + ", 1, 0), x" + J0 + "s = XV(" + J0 +
               ", -1, 0);\n";
        }
      }
      if (ch == 0)
        for (int k = 0; k < NT; ++k) c += "    double y" + std::to_string(k) + " = 0.0;\n";
      if (J->jouter) {  // stencils of the chunk in registers, x_j from shared memory
        const int i0 = ch * IC, i1 = std::min(NIN, (ch + 1) * IC);
        c += "    {\n";
        for (int i = i0; i < i1 && !dbg_nomath; ++i) {
          const std::string I0 = std::to_string(i - i0);
          c += "    const double k" + I0 + "d = K_D(" + I0 + "), k" + I0 + "e = K_E(" + I0 + "), k" + I0 + "w = K_W(" +
               I0 + "), k" + I0 + "n = K_N(" + I0 + "), k" + I0 + "s = K_S(" + I0 + ");\n";
        }
        for (int j : js) {
          if (dbg_nomath) break;
          std::string body;
          for (int i = i0; i < i1; ++i) {
            auto it = pairs.find({i, j});
            if (it == pairs.end()) continue;
            const std::string I0 = std::to_string(i - i0);
            body += "      { const double v = fma(k" + I0 + "d, xc, k" + I0 + "e * xe) + fma(k" + I0 + "w, xw, fma(k" + I0 +
                    "n, xn, k" + I0 + "s * xs));\n";
            for (auto& kc : it->second) {
              body += "        y" + std::to_string(kc.first) + " = fma(gcoef[" + std::to_string(J->coef.size()) +
                      "], v, y" + std::to_string(kc.first) + ");\n";
              J->coef.push_back(kc.second);
            }
            body += "      }\n";
          }
          if (body.empty()) continue;
          const std::string J0 = std::to_string(j);
          c += "    {\n      const double xc = XV(" + J0 + ", 0, 0), xe = XV(" + J0 + ", 0, 1), xw = XV(" + J0 +
               ", 0, -1), xn = XV(" + J0 + ", 1, 0), xs = XV(" + J0 + ", -1, 0);\n" + body + "    }\n";
        }
        c += "    }\n    STAGE_OUT();\n";
        continue;
      }
      // pairs of NI consecutive input terms at a time, their 5-FMA chains
      // interleaved term by term (independent chains hide the DFMA latency)
      std::vector<int> iis;
      for (int i = ch * IC; i < std::min(NIN, (ch + 1) * IC); ++i)
        if (i % GI == igrp) iis.push_back(i);
      for (size_t b = 0; b < iis.size() && !dbg_nomath; b += NI) {
        struct P { std::string ki, xj; const std::vector<std::pair<int, double>>* kc; };
        std::vector<P> ps;
        std::string kdecl;
        for (size_t u = b; u < std::min(iis.size(), b + NI); ++u) {
          const int i = iis[u];
          const std::string ii = std::to_string(i - ch * IC), K = "k" + std::to_string(u - b);
          bool any = false;
          for (int j : js) {
            auto it = pairs.find({i, j});
            if (it == pairs.end()) continue;
            ps.push_back({K, "x" + std::to_string(j), &it->second});
            any = true;
          }
          if (any)
            kdecl += "      const double " + K + "d = K_D(" + ii + "), " + K + "e = K_E(" + ii + "), " + K + "w = K_W(" + ii +
                     "), " + K + "n = K_N(" + ii + "), " + K + "s = K_S(" + ii + ");\n";
        }
        if (ps.empty()) continue;
        c += "    {\n" + kdecl;
        for (size_t q0 = 0; q0 < ps.size(); q0 += NIL) {
          const size_t q1 = std::min(ps.size(), q0 + NIL);
          std::string l0 = "      double", l1, l2, l3, l4, l5;
          for (size_t q = q0; q < q1; ++q) {
            const std::string v = "v" + std::to_string(q - q0), &k = ps[q].ki, &x = ps[q].xj;
            l0 += std::string(q == q0 ? " " : ", ") + v + " = " + k + "d * " + x + "c";
            l1 += "      " + v + " = fma(" + k + "e, " + x + "e, " + v + ");\n";
            l2 += "      " + v + " = fma(" + k + "w, " + x + "w, " + v + ");\n";
            l3 += "      " + v + " = fma(" + k + "n, " + x + "n, " + v + ");\n";
            l4 += "      " + v + " = fma(" + k + "s, " + x + "s, " + v + ");\n";
            for (auto& kc : *ps[q].kc) {
              const std::string cf = lit ? dlit(kc.second) : "gcoef[" + std::to_string(J->coef.size()) + "]";
              l5 += "      y" + std::to_string(kc.first) + " = fma(" + cf + ", " + v + ", y" + std::to_string(kc.first) +
                    ");\n";
              J->coef.push_back(kc.second);
            }
          }
          c += "      {\n" + l0 + ";\n" + l1 + l2 + l3 + l4 + l5 + "      }\n";
        }
        c += "    }\n";
      }
      c += "    STAGE_OUT();\n";
    }
    // mass on own terms (owner groups), then the fixed-order sum of the G partials
    auto emit_q = [&]() {
    // gamma M x2 on own terms, only when x2 is given (a uniform branch); inside,
    // predicated loads (no branches) so that all of them are in flight together
    for (int k : js) c += "    double q" + std::to_string(k) + " = 0.0;\n";
    c += "    if (A.x2 && valid) {\n";
    c += "      const double* x2p = A.x2 + it * A.xitem + (ll)gy * A.xpitch + gx;\n";
    c += "      const bool zE = gx + 1 < A.W, zW = gx > 0, zN = gy + 1 < A.H, zS = gy > 0;\n";
    for (int k : js) {
      const std::string K0 = std::to_string(k);
      c += "      { const double* p = x2p + " + K0 + " * A.xterm;\n";
      c += "        const double a0 = __ldg(p), a1 = zE ? __ldg(p + 1) : 0.0, a2 = zW ? __ldg(p - 1) : 0.0, "
           "a3 = zN ? __ldg(p + A.xpitch) : 0.0, a4 = zS ? __ldg(p - A.xpitch) : 0.0, "
           "a5 = (zN && zE) ? __ldg(p + A.xpitch + 1) : 0.0, a6 = (zS && zW) ? __ldg(p - A.xpitch - 1) : 0.0;\n";
      c += "        q" + K0 + " = fma(msw, a6, fma(mne, a5, fma(ms_, a4, fma(mn, a3, fma(mw, a2, fma(me, a1, md * a0)))))); }\n";
    }
    c += "    }\n";
    };
    if (owner && J->xg) {
    // mass stencil M [item][4][H][W] (diag, E, N, NE) from global memory
    c += "    const ll pl = (ll)A.W * A.H;\n";
    c += "    const double* mg = A.Mg + it * 4 * pl + (ll)(valid ? gy : 0) * A.W + (valid ? gx : 0);\n";
    c += "    const double md = valid ? __ldg(mg) : 0.0, me = valid ? __ldg(mg + pl) : 0.0, mw = hw ? __ldg(mg + pl - 1) : 0.0, "
         "mn = valid ? __ldg(mg + 2 * pl) : 0.0, ms_ = hs ? __ldg(mg + 2 * pl - A.W) : 0.0, "
         "mne = valid ? __ldg(mg + 3 * pl) : 0.0, msw = (hs && hw) ? __ldg(mg + 3 * pl - A.W - 1) : 0.0;\n";
    for (int k : js) {
      const std::string K0 = std::to_string(k);
      c += "    double m" + K0 + " = fma(md, x" + K0 + "c, fma(me, x" + K0 + "e, fma(mw, x" + K0 + "w, fma(mn, x" + K0 +
           "n, fma(ms_, x" + K0 + "s, fma(mne, XGV(" + K0 + ", 1, 1, hn && he), msw * XGV(" + K0 +
           ", -1, -1, hs && hw)))))));\n";
    }
    emit_q();
    }
    if (owner && !J->xg) {
    c += "    const double md = mb[ly * 32 + lane], me = mb[KOE + ly * 33 + lane + 1], mw = mb[KOE + ly * 33 + lane], "
         "mn = mb[MON + (ly + 1) * 32 + lane], ms_ = mb[MON + ly * 32 + lane], mne = mb[MONE + (ly + 1) * 33 + lane + 1], "
         "msw = mb[MONE + ly * 33 + lane];\n";
    c += "    const int gx = tx * 32 + lane, gy = ty * R + ly;\n";
    c += "    const bool valid = gx < A.W && gy < A.H;\n";
    for (int k : js) {
      const std::string K0 = std::to_string(k);
      if (J->jouter)
        c += "    double m" + K0 + " = fma(md, XV(" + K0 + ", 0, 0), fma(me, XV(" + K0 + ", 0, 1), fma(mw, XV(" + K0 +
             ", 0, -1), fma(mn, XV(" + K0 + ", 1, 0), fma(ms_, XV(" + K0 + ", -1, 0), fma(mne, XV(" + K0 +
             ", 1, 1), msw * XV(" + K0 + ", -1, -1)))))));\n";
      else
        c += "    double m" + K0 + " = fma(md, x" + K0 + "c, fma(me, x" + K0 + "e, fma(mw, x" + K0 + "w, fma(mn, x" + K0 +
             "n, fma(ms_, x" + K0 + "s, fma(mne, XV(" + K0 + ", 1, 1), msw * XV(" + K0 + ", -1, -1)))))));\n";
    }
    emit_q();
    } else if (!owner && !J->xg) {
      c += "    const int gx = tx * 32 + lane, gy = ty * R + ly;\n    (void)gx, (void)gy, (void)it;\n";
    }
    c += J->red_alias ? "    consumers_sync();  // everyone is done with xb (mass step) / red (previous tile)\n    double* red = xb;\n"
                      : "    consumers_sync();  // red of the previous tile is read\n    double* red = REDSEP;\n";
    if (G > 1) {
      for (int k = 0; k < NT; ++k) {
        const int own = grp[k];  // owner group of output k
        if (own == g) continue;
        const int slot = g < own ? g : g - 1;
        c += "    red[(" + std::to_string(slot) + " * NT + " + std::to_string(k) + ") * NODES + ly * 32 + lane] = y" +
             std::to_string(k) + ";\n";
      }
    }
    c += "    consumers_sync();\n";
    if (owner) c += "    if (valid) {\n      double* yo = A.y + it * A.yitem + (ll)gy * A.ypitch + gx;\n";
    for (int k : js) {
      if (!owner) break;
      const std::string K0 = std::to_string(k);
      std::string sum;
      for (int w = 0; w < G; ++w) {
        std::string term = w == g ? "y" + K0
                                  : "red[(" + std::to_string(w < g ? w : w - 1) + " * NT + " + K0 +
                                        ") * NODES + ly * 32 + lane]";
        sum = sum.empty() ? term : "(" + sum + " + " + term + ")";
      }
      c += "      yo[" + K0 + " * A.yterm] = fma(A.beta, " + sum + ", fma(A.alpha, m" + K0 + ", A.gamma * q" + K0 + "));\n";
    }
    if (owner) c += "    }\n";
    if (J->xg)
      c += "  }\n}\n#undef XGV\n";
    else
      c += "    __syncwarp();\n    if (lane == 0) mbar_arrive(XEMPTY(t & 1));  // x / M (and red) buffer free\n  }\n}\n";
    groups += c;
    dispatch += "    case " + std::to_string(g) + ": group" + std::to_string(g) + "(A, ly, lane, warp, mytiles, nst); break;\n";
  }
  dispatch += "  }";
  // timing experiment only (SGW_SGOP_DBG=2): every warp runs group 0's code (half the code footprint)
  if (std::getenv("SGW_SGOP_DBG") && std::atoi(std::getenv("SGW_SGOP_DBG")) == 2)
    dispatch.replace(dispatch.find("switch (gq)"), 11, "switch (0)");
  int pf = 0;  // measured: L2 prefetch beyond the ring does not help here
  if (const char* e = std::getenv("SGW_SGOP_PF")) pf = std::max(0, std::atoi(e));  // tuning hook
  int ef = 1;
  if (const char* e = std::getenv("SGW_SGOP_EF")) ef = std::atoi(e);  // tuning hook
  int ahead = J->S - 2;  // chunks in flight ahead of the one being consumed (warp 0 refills)
  if (const char* e = std::getenv("SGW_SGOP_AHEAD")) ahead = std::max(1, std::min(J->S - 1, std::atoi(e)));  // tuning hook
  std::string src = "#define AHEAD " + std::to_string(ahead) + "\n#define CPS " + std::to_string(J->cps) + "\n#define EF " + std::to_string(ef) + "\n#define PF " + std::to_string(pf) + "\n#define PROD " + std::to_string(J->prod) + "\n#define LA " + std::to_string(J->la) + "\n#define XG " + std::to_string(int(J->xg)) + "\n" + std::string("#define RED_ALIAS ") + (J->red_alias ? "1" : "0") + "\n#define NCOEF " + std::to_string(std::max<size_t>(1, J->coef.size())) +
                    "\n#define NT " + std::to_string(NT) + "\n#define NIN " + std::to_string(NIN) +
                    "\n#define R " + std::to_string(R) + "\n#define G " + std::to_string(G) + "\n#define IC " +
                    std::to_string(IC) + "\n#define S " + std::to_string(J->S) + "\n#define NCHUNK " +
                    std::to_string(J->NCHUNK) + "\n" + kDeviceTemplate;
  src.replace(src.find("@GROUPS@"), 8, groups);
  src.replace(src.find("@DISPATCH@"), 10, dispatch);
  if (const char* dump = std::getenv("SGW_SGOP_DUMP")) {
    if (FILE* f = std::fopen(dump, "w")) {
      std::fputs(src.c_str(), f);
      std::fclose(f);
    }
  }
  return src;
}

std::shared_ptr<SgOpJit> build_sgop(int NT, int NIN, const TensorHost& T) {
  auto J = std::make_shared<SgOpJit>();
  const std::string src = sgop_source(NT, NIN, T, J.get());
  if (src.empty()) return nullptr;
  const int R = J->R, G = J->G, IC = J->IC;
  // compile for sm_100a
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "sgop.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    throw Error(4, "nvrtcCreateProgram failed");
  const std::string regs = "--maxrregcount=" + std::to_string(J->regs);
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--fmad=true", regs.c_str()};
  const nvrtcResult rc = nvrtcCompileProgram(prog, 5, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, log.data());
    nvrtcDestroyProgram(&prog);
    throw Error(4, "SG operator JIT compile failed: " + log.substr(0, 2000));
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  std::string cubin(n, '\0');
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  SGW_CUDA(cudaLibraryLoadData(&J->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  SGW_CUDA(cudaLibraryGetKernel(&J->kern, J->lib, "sgop_kernel"));
  (void)R, (void)G, (void)IC;
  J->smem = size_t(sgop_smem_doubles(*J)) * 8;
  if (!J->coef.empty()) {  // c_ijk into the module's constant bank
    void* dptr = nullptr;
    size_t bytes = 0;
    SGW_CUDA(cudaLibraryGetGlobal(&dptr, &bytes, J->lib, "gcoef"));
    if (bytes < J->coef.size() * sizeof(double)) throw Error(4, "SG operator: coefficient table size mismatch");
    SGW_CUDA(cudaMemcpy(dptr, J->coef.data(), J->coef.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  SGW_CUDA(cudaFuncSetAttribute((const void*)J->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)J->smem));
  return J;
}

int sgop_rows(const SgOpJit& J) { return J.R; }

// x in the caller's layout -> [tile][NT][R+2][34] (the tile, one halo node
// around it; zeros outside the grid), each tile's block 128-byte aligned
__global__ void sgop_pack_x_kernel(const double* __restrict__ x, double* __restrict__ xt, long long xterm,
                                   long long xitem, int xpitch, int W, int H, int R, int NT, int tiles_x, int tiles_y,
                                   long long ntiles, long long xbuf) {
  const long long per = (long long)NT * (R + 2) * 34;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ntiles * per;
       e += (long long)gridDim.x * blockDim.x) {
    const long long tile = e / per;
    const int w = int(e % per), j = w / ((R + 2) * 34), rr = (w / 34) % (R + 2), cc = w % 34;
    const int tx = int(tile % tiles_x), ty = int((tile / tiles_x) % tiles_y), it = int(tile / ((long long)tiles_x * tiles_y));
    const int gy = ty * R - 1 + rr, gx = tx * 32 - 1 + cc;
    double v = 0.0;
    if (gy >= 0 && gy < H && gx >= 0 && gx < W) v = __ldg(x + it * xitem + j * xterm + (long long)gy * xpitch + gx);
    xt[tile * xbuf + w] = v;
  }
}

long long sgop_xt_doubles(const SgOpJit& J, const SgOpArgs& a) {
  const long long xbuf = ((long long)J.NT * (J.R + 2) * 34 + 15) / 16 * 16;
  return (long long)a.tiles_x * a.tiles_y * a.items * xbuf;
}

void sgop_tile_stencils(const SgOpJit& J, const double* K, const double* M, int W, int H, int items, int nin,
                        std::vector<double>& kt, std::vector<double>& mt, SgOpArgs& a) {
  const int R = J.R, tx_n = (W + 31) / 32, ty_n = (H + R - 1) / R;
  const long long kpi = (97LL * R + 33) / 2 * 2, mpi = (130LL * R + 66) / 2 * 2, plane = (long long)W * H;
  const long long ntiles = (long long)tx_n * ty_n * items;
  kt.assign(ntiles * nin * kpi, 0.0);
  mt.assign(ntiles * mpi, 0.0);
  auto at = [&](const double* P, long long pl, int r, int c) {
    return (r >= 0 && r < H && c >= 0 && c < W) ? P[pl * plane + (long long)r * W + c] : 0.0;
  };
  for (long long tile = 0; tile < ntiles; ++tile) {
    const int tx = int(tile % tx_n), ty = int((tile / tx_n) % ty_n), it = int(tile / ((long long)tx_n * ty_n));
    const int r0 = ty * R, c0 = tx * 32;
    for (int i = 0; i < nin; ++i) {
      double* d = &kt[(tile * nin + i) * kpi];
      const long long pl = ((long long)it * nin + i) * 3;
      for (int rr = 0; rr < R; ++rr)
        for (int cc = 0; cc < 32; ++cc) d[rr * 32 + cc] = at(K, pl, r0 + rr, c0 + cc);
      for (int rr = 0; rr < R; ++rr)
        for (int cc = 0; cc < 33; ++cc) d[32 * R + rr * 33 + cc] = at(K, pl + 1, r0 + rr, c0 - 1 + cc);
      for (int rr = 0; rr <= R; ++rr)
        for (int cc = 0; cc < 32; ++cc) d[65 * R + rr * 32 + cc] = at(K, pl + 2, r0 - 1 + rr, c0 + cc);
    }
    double* m = &mt[tile * mpi];
    const long long pm = (long long)it * 4;
    for (int rr = 0; rr < R; ++rr)
      for (int cc = 0; cc < 32; ++cc) m[rr * 32 + cc] = at(M, pm, r0 + rr, c0 + cc);
    for (int rr = 0; rr < R; ++rr)
      for (int cc = 0; cc < 33; ++cc) m[32 * R + rr * 33 + cc] = at(M, pm + 1, r0 + rr, c0 - 1 + cc);
    for (int rr = 0; rr <= R; ++rr)
      for (int cc = 0; cc < 32; ++cc) m[65 * R + rr * 32 + cc] = at(M, pm + 2, r0 - 1 + rr, c0 + cc);
    for (int rr = 0; rr <= R; ++rr)
      for (int cc = 0; cc < 33; ++cc) m[97 * R + 32 + rr * 33 + cc] = at(M, pm + 3, r0 - 1 + rr, c0 - 1 + cc);
  }
  a.W = W, a.H = H, a.tiles_x = tx_n, a.tiles_y = ty_n, a.items = items;
}

bool sgop_packs_x(const SgOpJit& J) { return !J.xg; }

void launch_sgop(const SgOpJit& J, const SgOpArgs& a, cudaStream_t st) {
  const int tiles = a.tiles_x * a.tiles_y * a.items;
  if (!J.xg) {
    const long long xbuf = ((long long)J.NT * (J.R + 2) * 34 + 15) / 16 * 16;
    const long long tot = (long long)tiles * J.NT * (J.R + 2) * 34;
    sgop_pack_x_kernel<<<(unsigned)std::min<long long>((tot + 255) / 256, 8 * kNumSMs * 4), 256, 0, st>>>(
        a.x, const_cast<double*>(a.xt), a.xterm, a.xitem, a.xpitch, a.W, a.H, J.R, J.NT, a.tiles_x, a.tiles_y, tiles,
        xbuf);
    SGW_LAUNCHED();
  }
  const int grid = std::max(1, std::min(tiles, J.cps * kNumSMs));
  void* args[] = {const_cast<SgOpArgs*>(&a)};
  SGW_CUDA(cudaLaunchKernel((const void*)J.kern, dim3(grid), dim3(32 * (J.R * J.G + J.prod)), args, J.smem, st));
  SGW_LAUNCHED();
}

}  // namespace sgw
