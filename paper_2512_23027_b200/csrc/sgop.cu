// Fused stochastic-Galerkin operator apply (src/sg.cpp:425-447):
//   y_k = alpha M x_k + beta sum_{(i,j)} c_ijk K_i x_j
// on the reduced (nx-1) x (ny-1) dof grid.  The kernel is generated and
// compiled at setup (NVRTC, sm_100a) for the solver's triple-product tensor.
//
// Stored operator: two couplings per node and input term.  Every row of a
// P1 stiffness matrix sums to zero (the element grad-grad matrix annihilates
// constants; src/sg.cpp:60-78) and on this mesh the hypotenuse couplings are
// identically zero, so with x = 0 on the Dirichlet boundary
//   (K_i x)(p) = sum_{d in E,W,N,S} k_i^d(p) (x(p+d) - x(p))
// where k^W(p) = k^E(p-1) and k^S(p) = k^N(p-row).  The couplings of a row to
// the (removed) boundary nodes are recovered from the reduced diagonal:
// sum_missing = -(K_pp + sum_present).  So the kernel streams 2 values per
// node and term (east, north) instead of 3, and spends 4 flops-ops per (i, j)
// pair instead of 5.
//
//   * One thread per node (a team of G warps per row when the register file
//     cannot hold every term): the 4 differences of every x_j it owns (scaled
//     by beta) and all P+1 outputs live in registers; per input term i the
//     thread reads its 4 couplings from shared memory and runs the generated
//     straight-line (i, j) pair code with c_ijk as literals.
//   * Teams are independent pipelines: each streams its own grid rows through
//     its own S-stage ring of 1-D TMA bulk copies (mbarrier transaction
//     counts, evict-first), one stage = one chunk of IC input terms of one row
//     (2 copies: the row's coupling blocks and the south row's), and refills a
//     stage as soon as it has consumed it.  No CTA-wide synchronisation in the
//     main loop, so a team that waits for its x loads does not hold up others.
//   * Work split: the 32-node grid rows of all strips, in one linear order, are
//     divided evenly over the CTAs (one row granularity); inside a CTA the
//     (row, chunk) units are divided evenly over the teams, so every SM and
//     every team gets the same bytes and flops.  A row split between teams is
//     summed from the pieces' partials in team order at the end (bitwise
//     reproducible); the piece that starts a row adds the mass term.
//   * The G partial outputs of a node are summed in shared memory in fixed
//     group order.
// Layout of the stored couplings K (built by sgop_pack_stencils):
//   [strip][y + 1 (rows -1..H-1)][i][ E columns -1..31 (33) | 0 | N columns 0..31 (32) ]
#include <nvrtc.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <string>

#include "solver.cuh"

namespace sgw {

namespace {
const char* kDeviceTemplate = R"CUDA(
typedef long long ll;
struct SgOpArgs {
  const double* K; const double* x; double* y; double* part;
  ll xterm, yterm;
  int W, H, xpitch, ypitch, strips, pad_;
  double alpha, beta, md, mo;
};
#define NTHR (32 * NW)
#define KB 66                        /* doubles per (grid row, input term) block: E 33 | pad | N 32 */
#define STG ((RP + 1) * IC * KB)     /* stage: rows row-1 .. row+RP-1 of one chunk */
extern __shared__ __align__(1024) double sm[];
#define XROWS (RP + 2)
#define XN (NT * XROWS * 34)         /* x of a pass: rows row-1 .. row+RP, columns -1..32 of the strip */
#define XBUF ((XN + 15) / 16 * 16)
#define RING (sm)
#define XS (sm + S * STG)
#define RED (sm + S * STG + XBUF)
#define FULL(i) ((unsigned long long*)(sm + S * STG + XBUF + REDN) + (i))
#define KCNT(i) ((int*)((unsigned long long*)(sm + S * STG + XBUF + REDN) + S) + (i))

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk(double* s, const double* g, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(su(s)), "l"(g), "r"(bytes), "r"(su(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(su(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(su(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
               :: "r"(su(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" :: "n"(NW * 32) : "memory"); }

__device__ __forceinline__ void cp8(double* s, const double* g, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" :: "r"(su(s)), "l"(g), "r"(ok ? 8 : 0) : "memory");
}

/* pass starting at linear row p of a CTA range ending at r1 */
__device__ __forceinline__ void pass_at(const SgOpArgs& A, int p, int r1, int& strip, int& row, int& rows) {
  strip = p / A.H, row = p - strip * A.H;
  rows = min(RP, min(A.H - row, r1 - p));
}

/* stage q (pass q / NCHUNK, chunk q % NCHUNK) of the CTA's range: one bulk copy
   of the chunk's blocks of rows row-1 .. row+rows-1 */
__device__ __forceinline__ void issue(const SgOpArgs& A, int r0, int r1, int q, int pass_hint, int p_hint) {
  int pass = q / NCHUNK, p = p_hint, strip, row, rows;
  for (int k = pass_hint; ; ++k) {
    if (p >= r1) return;
    pass_at(A, p, r1, strip, row, rows);
    if (k == pass) break;
    p += rows;
  }
  const int ch = q % NCHUNK, i0 = ch * IC, ni = min(IC, NIN - i0);
  /* K[strip][chunk][y + 1][ni][KB]: the chunk's rows are contiguous */
  const double* src = A.K + ((ll)strip * NIN * (A.H + 1) + (ll)i0 * (A.H + 1) + (ll)row * ni) * KB;
  const unsigned bytes = (unsigned)((rows + 1) * ni * KB * 8);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(FULL(q % S), bytes);
  bulk(RING + (q % S) * STG, src, bytes, FULL(q % S));
}

/* x of the pass starting at row p into XS (asynchronous copies, zeros
   outside the grid): issued while the previous pass computes */
__device__ __forceinline__ void xload(const SgOpArgs& A, int p, int r1) {
  if (p < r1) {
    int strip, row, rows;
    pass_at(A, p, r1, strip, row, rows);
    /* warp w copies row segments w, w + NW, ... (segment = (term, tile row));
       lane l columns l and 32 + l (l < 2) */
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, x0 = strip * 32 - 1 + lane;
    const bool c0 = x0 >= 0 && x0 < A.W, c1 = lane < 2 && x0 + 32 < A.W;
    int j = warp / XROWS, rr = warp - j * XROWS;
    for (int seg = warp; seg < NT * XROWS; seg += NW) {
      const int yy = row - 1 + rr;
      const bool ry = rr <= rows + 1 && yy >= 0 && yy < A.H;
      const double* src = A.x + j * A.xterm + (ll)yy * A.xpitch + x0;
      double* dst = XS + seg * 34 + lane;
      cp8(dst, ry && c0 ? src : A.x, ry && c0);
      if (lane < 2) cp8(dst + 32, ry && c1 ? src + 32 : A.x, ry && c1);
      rr += NW;
      while (rr >= XROWS) rr -= XROWS, ++j;
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
#define XV(j, dr, dc) XS[((j) * XROWS + ly + 1 + (dr)) * 34 + lane + 1 + (dc)]

/* couplings of input term u (of NI in the chunk) of the current stage: own
   east / west (= east of the west neighbour) / own north / south (= north of
   the south neighbour) */
#define KE(u, NI) kb[(((ly) + 1) * (NI) + (u)) * KB + lane + 1]
#define KW(u, NI) kb[(((ly) + 1) * (NI) + (u)) * KB + lane]
#define KN(u, NI) kb[(((ly) + 1) * (NI) + (u)) * KB + 34 + lane]
#define KS(u, NI) kb[((ly) * (NI) + (u)) * KB + 34 + lane]

@GROUPS@

extern "C" __global__ void __launch_bounds__(NTHR, CPS) sgop_kernel(const SgOpArgs A) {
  const int tot = A.strips * A.H;
  const int r0 = (int)((ll)tot * blockIdx.x / gridDim.x), r1 = (int)((ll)tot * (blockIdx.x + 1) / gridDim.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(FULL(i), 1), *KCNT(i) = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < S && !DBG2; ++i) issue(A, r0, r1, i, 0, r0);
  }
  xload(A, r0, r1);
  __syncthreads();
  const int ly = warp / G, gq = warp % G;
  int q = 0, pass = 0;
  for (int p = r0; p < r1; ++pass) {
    int strip, row, rows;
    pass_at(A, p, r1, strip, row, rows);
    const bool act = ly < rows;
    const int y = row + ly, x = strip * 32 + lane;
    @DISPATCH@
    p += rows;
  }
}
)CUDA";

std::string dlit(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  std::string s(b);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
}  // namespace

struct SgOpJit {
  int NT = 0, NIN = 0, G = 1, RP = 8, NW = 8, IC = 8, S = 3, NCHUNK = 0, CPS = 1, regs = 255;
  long long n_pairs = 0, n_coef = 0;  // distinct (i, j) with some c_ijk != 0; full (i, j, k) entries
  size_t smem = 0;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  ~SgOpJit() {
    if (lib) cudaLibraryUnload(lib);
  }
};

static constexpr int kBlock = 66;  // doubles per (grid row, input term) block: E 33 | pad | N 32
static long long red_doubles(const SgOpJit& J) { return J.G > 1 ? (long long)(J.G - 1) * J.NT * J.RP * 32 : 0; }
static long long x_doubles(const SgOpJit& J) { return ((long long)J.NT * (J.RP + 2) * 34 + 15) / 16 * 16; }

// CUDA source of the operator specialised for (NT, NIN, T); fills J's shape.
// Returns "" when the basis is too large for register-resident terms (the
// caller then uses the table-driven kernel in step.cu).
std::string sgop_source(int NT, int NIN, const TensorHost& T, SgOpJit* J) {
  J->NT = NT, J->NIN = NIN;
  // 32-bit registers per thread: 4 differences per owned input term j and
  // every output k (doubles: 2 registers each), plus addresses, couplings and
  // chains.  Eight warps per CTA (NW a multiple of 4 keeps the register file
  // evenly split over the SM sub-partitions): G groups x RP = 8 / G rows.
  auto regs = [&](int g) { return 2 * (4 * ((NT + g - 1) / g) + NT) + 34; };
  int G = 1;
  while (G < 8 && regs(G) > 240) G *= 2;
  G = env_int("SGW_SGOP_G", G);  // tuning hook
  if (regs(G) > 255 || G > 8) return std::string();
  J->G = G;
  // rows per pass: 8 warps (G = 1, 2); 12 warps for G = 4 (measured at C3:
  // 0.79 vs 1.01 ms with 8 warps, despite ptxas's 168-register cap)
  J->RP = std::max(1, env_int("SGW_SGOP_RP", G == 4 && regs(G) <= 180 ? 3 : 8 / G));  // tuning hook
  J->NW = J->RP * G;
  const int nthr = 32 * J->NW;
  J->CPS = std::max(1, std::min(4, 65536 / (nthr * std::max(64, regs(G)))));
  J->CPS = std::max(1, env_int("SGW_SGOP_CPS", J->CPS));  // tuning hook
  J->regs = std::min(255, (65536 / (nthr * J->CPS)) & ~7);
  // stages of (RP + 1) x IC blocks; about 6 of them in the shared memory
  const long long budget = (227LL * 1024 / J->CPS - 1024) / 8 - red_doubles(*J) - x_doubles(*J);
  const long long row_term = (long long)(J->RP + 1) * kBlock;
  J->IC = int(std::max(1LL, std::min<long long>(NIN, budget / 3 / row_term)));  // measured: 3 deep stages beat 4-6 shallower
  J->IC = std::max(1, std::min(NIN, env_int("SGW_SGOP_IC", J->IC)));  // tuning hook
  J->NCHUNK = (NIN + J->IC - 1) / J->IC;
  J->S = int(std::max(2LL, std::min<long long>(12, budget / (J->IC * row_term))));
  J->S = std::max(2, env_int("SGW_SGOP_S", J->S));  // tuning hook
  // full (i, j) -> [(k, c)] expansion of the j <= k tensor (pce.hpp:24-40)
  std::map<std::pair<int, int>, std::vector<std::pair<int, double>>> pairs;
  for (size_t e = 0; e < T.v.size(); ++e) {
    pairs[{T.i[e], T.j[e]}].push_back({T.k[e], T.v[e]});
    if (T.j[e] != T.k[e]) pairs[{T.i[e], T.k[e]}].push_back({T.j[e], T.v[e]});
  }
  J->n_pairs = (long long)pairs.size();
  J->n_coef = 0;
  for (auto& p : pairs) J->n_coef += (long long)p.second.size();
  // j groups balanced by work (4 ops per pair + 1 per coefficient)
  std::vector<long long> wj(NT, 0);
  for (auto& p : pairs) wj[p.first.second] += 4 + (long long)p.second.size();
  std::vector<int> order(NT), grp(NT, 0);
  for (int j = 0; j < NT; ++j) order[j] = j;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return wj[a] > wj[b]; });
  std::vector<long long> load(G, 0);
  std::vector<int> cnt(G, 0);
  const int cap = (NT + G - 1) / G;
  for (int j : order) {
    int g = -1;
    for (int c = 0; c < G; ++c)
      if (cnt[c] < cap && (g < 0 || load[c] < load[g])) g = c;
    grp[j] = g, load[g] += wj[j], ++cnt[g];
  }
  const int NIL = std::max(1, env_int("SGW_SGOP_NIL", 4));  // pair chains interleaved
  const std::string call = "(A, r0, r1, q, pass, p, rows, act, x, y, ly, lane);";
  std::string groups, dispatch = G == 1 ? "group0" + call : "switch (gq) {\n";
  for (int g = 0; g < G; ++g) {
    std::vector<int> js;
    for (int j = 0; j < NT; ++j)
      if (grp[j] == g) js.push_back(j);
    std::string c;
    c += "__device__ __forceinline__ void group" + std::to_string(g) +
         "(const SgOpArgs& A, int r0, int r1, int& q, int pass, int p0, int rows, bool act, int x, int y, int ly, int lane) {\n";
    c += "  const bool valid = act && x < A.W;\n";
    c += "  asm volatile(\"cp.async.wait_all;\" ::: \"memory\");\n  consumers_sync();  // this pass's x is in XS\n";
    for (int k = 0; k < NT; ++k)
      if (grp[k] != g) c += "  double y" + std::to_string(k) + " = 0.0;\n";
    for (int j : js) {
      const std::string J0 = std::to_string(j);
      c += "  double y" + J0 + ", d" + J0 + "e, d" + J0 + "w, d" + J0 + "n, d" + J0 + "s;\n";
      c += "  {\n";
      c += "    const double c = XV(" + J0 + ", 0, 0), e = XV(" + J0 + ", 0, 1), w = XV(" + J0 + ", 0, -1), n = XV(" + J0 +
           ", 1, 0), s = XV(" + J0 + ", -1, 0), ne = XV(" + J0 + ", 1, 1), sw = XV(" + J0 + ", -1, -1);\n";
      c += "    y" + J0 + " = A.alpha * fma(A.md, c, A.mo * (((e + w) + (n + s)) + (ne + sw)));\n";
      c += "    d" + J0 + "e = A.beta * (e - c), d" + J0 + "w = A.beta * (w - c), d" + J0 + "n = A.beta * (n - c), d" + J0 +
           "s = A.beta * (s - c);\n  }\n";
    }
    c += "  consumers_sync();  // XS is read: prefetch the next pass's x\n  xload(A, p0 + rows, r1);\n";
    // chunk loop at run time (one release / refill site), the chunk's pair code
    // behind a switch
    // timing experiments only: SGW_SGOP_DBG=1 streams without the math, 2 runs
    // the math on whatever the ring holds without streaming
    const int dbg = env_int("SGW_SGOP_DBG", 0);
    c += "  for (int ch = 0; ch < NCHUNK; ++ch, ++q) {\n";
    if (dbg != 2) c += "    mbar_wait(FULL(q % S), (unsigned)(q / S) & 1u);\n";
    c += "    const double* kb = RING + (q % S) * STG;\n    if (act" + std::string(dbg == 1 ? " && A.W < 0" : "") + ") switch (ch) {\n";
    for (int ch = 0; ch < J->NCHUNK; ++ch) {
      c += "    case " + std::to_string(ch) + ": {\n";
      const int i0 = ch * J->IC, i1 = std::min(NIN, i0 + J->IC);
      const std::string NI = std::to_string(i1 - i0);
      for (int i = i0; i < i1; ++i) {
        struct P { std::string j; const std::vector<std::pair<int, double>>* kc; };
        std::vector<P> ps;
        for (int j : js) {
          auto it = pairs.find({i, j});
          if (it != pairs.end()) ps.push_back({std::to_string(j), &it->second});
        }
        if (ps.empty()) continue;
        const std::string u = std::to_string(i - i0) + ", " + NI;
        c += "      {\n      const double ke = KE(" + u + "), kw = KW(" + u + "), kn = KN(" + u + "), ks = KS(" + u + ");\n";
        for (size_t q0 = 0; q0 < ps.size(); q0 += NIL) {
          const size_t q1 = std::min(ps.size(), q0 + NIL);
          std::string l0 = "      double", l1, l2, l3, l4;
          for (size_t qq = q0; qq < q1; ++qq) {
            const std::string v = "v" + std::to_string(qq - q0), &j = ps[qq].j;
            l0 += std::string(qq == q0 ? " " : ", ") + v + " = ke * d" + j + "e";
            l1 += "      " + v + " = fma(kw, d" + j + "w, " + v + ");\n";
            l2 += "      " + v + " = fma(kn, d" + j + "n, " + v + ");\n";
            l3 += "      " + v + " = fma(ks, d" + j + "s, " + v + ");\n";
            for (auto& kc : *ps[qq].kc)
              l4 += "      y" + std::to_string(kc.first) + " = fma(" + dlit(kc.second) + ", " + v + ", y" +
                    std::to_string(kc.first) + ");\n";
          }
          c += "      {\n" + l0 + ";\n" + l1 + l2 + l3 + l4 + "      }\n";
        }
        c += "      }\n";
      }
      c += "    } break;\n";
    }
    c += "    }\n    __syncwarp();\n";
    if (dbg != 2)
      c += "    if (lane == 0) {\n      __threadfence_block();\n"
           "      if (atomicAdd(KCNT(q % S), 1) == NW - 1) {  // the last warp to release the stage refills it\n"
           "        *KCNT(q % S) = 0;\n        issue(A, r0, r1, q + S, pass, p0);\n      }\n    }\n";
    c += "  }\n";
    if (G > 1) {
      c += "  consumers_sync();  // the previous pass's partials are read\n  if (act) {\n";
      for (int k = 0; k < NT; ++k) {
        const int own = grp[k];
        if (own == g) continue;
        const int slot = g < own ? g : g - 1;
        c += "    RED[(" + std::to_string(slot) + " * NT + " + std::to_string(k) + ") * (RP * 32) + ly * 32 + lane] = y" +
             std::to_string(k) + ";\n";
      }
      c += "  }\n  consumers_sync();\n";
    }
    c += "  if (valid) {\n    double* yo = A.y + (ll)y * A.ypitch + x;\n";
    for (int k : js) {
      const std::string K0 = std::to_string(k);
      std::string sum;
      for (int w = 0; w < G; ++w) {
        const std::string term = w == g ? "y" + K0
                                        : "RED[(" + std::to_string(w < g ? w : w - 1) + " * NT + " + K0 +
                                              ") * (RP * 32) + ly * 32 + lane]";
        sum = sum.empty() ? term : "(" + sum + " + " + term + ")";
      }
      c += "    yo[" + K0 + " * A.yterm] = " + sum + ";\n";
    }
    c += "  }\n}\n";
    groups += c;
    if (G > 1) dispatch += "    case " + std::to_string(g) + ": group" + std::to_string(g) + call + " break;\n";
  }
  if (G > 1) dispatch += "    }";
  std::string src = "#define NT " + std::to_string(NT) + "\n#define NIN " + std::to_string(NIN) + "\n#define G " +
                    std::to_string(G) + "\n#define RP " + std::to_string(J->RP) + "\n#define NW " +
                    std::to_string(J->NW) + "\n#define IC " + std::to_string(J->IC) + "\n#define NCHUNK " +
                    std::to_string(J->NCHUNK) + "\n#define S " + std::to_string(J->S) + "\n#define CPS " +
                    std::to_string(J->CPS) + "\n#define REDN " + std::to_string(red_doubles(*J)) + "\n#define DBG2 " +
                    std::to_string(int(env_int("SGW_SGOP_DBG", 0) == 2)) + "\n" +
                    kDeviceTemplate;
  src.replace(src.find("@GROUPS@"), 8, groups);
  src.replace(src.find("@DISPATCH@"), 10, dispatch);
  J->smem = size_t(J->S * (J->RP + 1) * J->IC * kBlock + x_doubles(*J) + red_doubles(*J)) * 8 + size_t(J->S) * 12 + 16;
  if (const char* dump = std::getenv("SGW_SGOP_DUMP")) {
    if (FILE* f = std::fopen(dump, "w")) {
      std::fputs(src.c_str(), f);
      std::fclose(f);
    }
  }
  return src;
}

std::shared_ptr<SgOpJit> build_sgop(int NT, int NIN, const TensorHost& T) {
  if (env_int("SGW_SGOP_OFF", 0)) return nullptr;  // tuning hook: table-driven kernel only
  auto J = std::make_shared<SgOpJit>();
  const std::string src = sgop_source(NT, NIN, T, J.get());
  if (src.empty()) return nullptr;
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
  SGW_CUDA(cudaFuncSetAttribute((const void*)J->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)J->smem));
  return J;
}

// Couplings of the reduced global stencils Kg [i][3][H][W] (diag, E, N; host.cpp
// build_stencils) in the operator's block layout K[strip][chunk][y + 1][i][66]:
// E of columns -1..31 of the strip, a zero pad, N of columns 0..31 (row y = -1
// holds the south boundary slots).  Returns false (operator not usable) when
// the mass stencil Mg [4][H][W] is not the constant one of the structured mesh.
bool sgop_pack_stencils(const SgOpJit& J, const double* Kg, const double* Mg, int W, int H, int nin,
                        std::vector<double>& kt, SgOpArgs& a) {
  const long long n = (long long)W * H;
  // constant mass stencil: diag md, E / N / NE couplings mo (interior couplings)
  const double md = Mg[0];
  double mo = 0.0;
  bool have_mo = false;
  for (long long d = 0; d < n; ++d) {
    const int x = int(d % W), y = int(d / W);
    if (std::fabs(Mg[d] - md) > 1e-13 * std::fabs(md)) return false;
    const bool ok[3] = {x + 1 < W, y + 1 < H, x + 1 < W && y + 1 < H};
    for (int c = 0; c < 3; ++c) {
      if (!ok[c]) continue;
      const double v = Mg[(c + 1) * n + d];
      if (!have_mo) mo = v, have_mo = true;
      if (std::fabs(v - mo) > 1e-13 * std::fabs(md)) return false;
    }
  }
  const int strips = (W + 31) / 32;
  kt.assign(size_t(strips) * (H + 1) * nin * kBlock, 0.0);
  std::vector<double> miss(n);  // the couplings of a row to removed boundary nodes, summed
  for (int i = 0; i < nin; ++i) {
    const double* D = Kg + (size_t(i) * 3) * n;
    const double *E = D + n, *N = D + 2 * n;
    for (long long d = 0; d < n; ++d) {
      const int x = int(d % W), y = int(d / W);
      double s = D[d];
      if (x + 1 < W) s += E[d];
      if (x > 0) s += E[d - 1];
      if (y + 1 < H) s += N[d];
      if (y > 0) s += N[d - W];
      miss[d] = -s;
    }
    // chunk-major: K[strip][chunk][y + 1][term of the chunk][66]
    const int i0 = i / J.IC * J.IC, ni = std::min(J.IC, nin - i0);
    // each row's missing couplings go to its first missing slot in the order
    // west, south, east, north (every slot is read by that row only)
    for (int st = 0; st < strips; ++st)
      for (int r = 0; r <= H; ++r) {
        double* b = &kt[((size_t(st) * nin * (H + 1) + size_t(i0) * (H + 1) + size_t(r) * ni) + (i - i0)) * kBlock];
        const int y = r - 1;
        for (int c = 0; c < 33 && y >= 0; ++c) {
          const int x = st * 32 - 1 + c;
          double v = 0.0;
          if (x >= 0 && x + 1 < W) v = E[(long long)y * W + x];
          else if (x == -1) v = miss[(long long)y * W];        // west slot of (0, y)
          else if (x == W - 1 && W > 1 && y > 0) v = miss[(long long)y * W + x];  // east slot
          b[c] = v;
        }
        for (int c = 0; c < 32; ++c) {
          const int x = st * 32 + c;
          if (x >= W) continue;
          double v = 0.0;
          if (y >= 0 && y + 1 < H) v = N[(long long)y * W + x];
          else if (y == -1 && x > 0) v = miss[x];  // south slot of (x, 0) (x = 0: the west slot has it)
          else if (y == H - 1 && y >= 0 && x > 0 && x + 1 < W && H > 1) v = miss[(long long)y * W + x];  // north slot
          b[34 + c] = v;
        }
      }
  }
  a.K = nullptr;
  a.W = W, a.H = H, a.strips = strips;
  a.md = md, a.mo = mo;
  (void)J;
  return true;
}

long long sgop_scratch_doubles(const SgOpJit&, int, int) { return 1; }

void launch_sgop(const SgOpJit& J, const SgOpArgs& a, cudaStream_t st) {
  const long long rows = (long long)a.strips * a.H;
  const int grid = int(std::max(1LL, std::min<long long>(rows, (long long)J.CPS * kNumSMs)));
  void* args[] = {const_cast<SgOpArgs*>(&a)};
  SGW_CUDA(cudaLaunchKernel((const void*)J.kern, dim3(grid), dim3(32 * J.NW), args, J.smem, st));
  SGW_LAUNCHED();
}

double sgop_flops(const SgOpJit& J, long long n) {
  // per node: 4 ops per (i, j) pair, 1 FMA per c_ijk, 7 per mass row (FMA = 2 flops)
  return 2.0 * double(n) * (4.0 * J.n_pairs + J.n_coef + 7.0 * J.NT);
}

}  // namespace sgw
