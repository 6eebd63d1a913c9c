// GPU SG solver: device-resident data of the interface-Schur PCG / NN2 path.
//
// Data layout in HBM (all fp64):
//  * global state u, v, a, um, uc: term-major [j * n + d] (reference layout,
//    src/sg.cpp:362-365).
//  * global interface vectors: term-major [j * n_iface + q] (src/dd.cpp:86).
//  * local interface vectors ("LI" buffers): per subdomain s a padded slice
//    [li_off[s], li_off[s] + 64 * nt_S[s]) holding [j * ng_s + p].
//  * S_s and Q_s = S_rr^-1: lower 64x64 tiles, row-major inside a tile,
//    diagonal tiles stored full (TilePack).
//  * Psi_s = S_rr^-1 S_rc: column-major r_s x c_s.  F_cc^-1: n_C x n_C.
//  * interior solve: block-tridiagonal by interior grid rows, block B =
//    W (P+1) (node-major, term-minor); per grid row the lower tiles of
//    D_k^-1 = (L_kk L_kk^T)^-1 and the S/SW coupling band of A_{k+1,k} in
//    both orientations (sweep.cu).  Setup copies Linv[s][k] = L_kk^-1 and
//    Lsub[s][k] = A_{k+1,k} -> L_{k+1,k} are dense column-major B x B.
#pragma once

#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <memory>
#include <vector>

#include "comm.hpp"
#include "common.cuh"
#include "host.hpp"
#include "tiles.cuh"

namespace sgw {

struct SweepLayout;

// Arguments of the JIT-compiled SG operator (sgop.cu); identical layout to the
// device-side struct in the generated source.
struct SgOpArgs {
  const double* K;  // couplings in block layout (sgop_pack_stencils)
  const double* x;
  double* y;
  double* part;  // partial rows scratch (sgop_scratch_doubles)
  long long xterm, yterm;
  int W, H, xpitch, ypitch, strips, pad_;
  double alpha, beta, md, mo;  // y = alpha M x + beta K x; constant mass stencil (diag, off-diagonal)
};
struct SgOpJit;
// nullptr when the basis is too large for the register-resident kernel
std::shared_ptr<SgOpJit> build_sgop(int NT, int NIN, const TensorHost& T);
void launch_sgop(const SgOpJit& J, const SgOpArgs& a, cudaStream_t st);
double sgop_flops(const SgOpJit& J, long long n);
// Strip-major couplings of the reduced stencils Kg [i][3][H][W]; false when the
// mass stencil Mg [4][H][W] is not constant (the kernel assumes it is).
bool sgop_pack_stencils(const SgOpJit& J, const double* Kg, const double* Mg, int W, int H, int nin,
                        std::vector<double>& kt, SgOpArgs& a);
long long sgop_scratch_doubles(const SgOpJit& J, int W, int H);

// device bytes held by every DBuf of the process (all element types)
struct DevBytes {
  static inline std::atomic<long long> total{0};
};

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { reset(); }
  void alloc(size_t count) {
    reset();
    n = count;
    if (count) {
      cudaError_t e = cudaMalloc(&p, count * sizeof(T));
      if (e != cudaSuccess) {
        p = nullptr;
        throw Error(6, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed");
      }
      DevBytes::total += count * sizeof(T);
    }
  }
  void upload(const std::vector<T>& h) {
    alloc(h.size());
    if (!h.empty()) SGW_CUDA(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
  void zero(cudaStream_t st) {
    if (n) SGW_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), st));
  }
  void reset() {
    if (p) {
      cudaFree(p);
      DevBytes::total -= n * sizeof(T);
    }
    p = nullptr;
    n = 0;
  }
};

// Batch of symmetric matrices stored as lower 64x64 tiles.
// llt_regularized (src/dd.cpp:66-76) + explicit inverse of an SPD n x n
// column-major device matrix, in place (setup.cu)
void spd_inverse(cusolverDnHandle_t sol, cudaStream_t st, double* A, int n, DBuf<double>& work, DBuf<int>& info,
                 const char* what);

struct TilePack {
  int nmat = 0;
  std::vector<int> dim, ntile;       // per matrix: dimension, tiles per side
  std::vector<long long> tile_base;  // first tile of each matrix
  std::vector<long long> xoff;       // padded local-vector offset (64 * sum ntile)
  long long n_tiles = 0, xlen = 0;
  DBuf<int4> desc;  // per tile: {matrix, I, J, unused}
  DBuf<int2> tx;    // per tile: local-vector offsets of the I and J segments
  DBuf<double> tiles, rowpart, colpart;
  DBuf<long long> d_tile_base, d_xoff;
  DBuf<int> d_ntile, d_dim;
  void plan(const std::vector<int>& dims, bool alloc_tiles = true);
  long long bytes() const { return n_tiles * kTile * kTile * 8; }
};

// Contiguous per-CTA tile ranges of a TilePack for the persistent PCG kernel
// (pcg_fused.cu RangePack): CTA c walks tiles [t_first[c], t_first[c + 1]).
struct RangeBufs {
  DBuf<long long> t_first, pbase;
  DBuf<int4> start;
  DBuf<int> c0, ncta;
  DBuf<double> part;
  std::vector<long long> h_pbase;  // host copies (scatter descriptors)
  std::vector<int> h_ncta;
  void plan(const std::vector<long long>& tile_base, const std::vector<int>& nI, const std::vector<int>& nJ, int grid);
};

// G tensor lists by output term k: entries (i, j, g) in for_each order.
struct GList {
  const int *ptr, *i, *j;
  const double* v;
};
// Kernel-side view of the per-subdomain local operator data.
struct LocalArgs {
  const double *Kl, *Ml;
  GList g;
  const int* lid_to_p;
  const long long* lioff;
  const int* ng;
  const int* sub_gid;  // local subdomain -> global id (row-major)
  int nl, nin, nt, mx, my, px, nx, py, ny, H, B;
  double ms, ss;
};

struct Timers {
  double pcg_ms = 0, step_ms = 0, rhs_ms = 0, rec_ms = 0;
  long long iterations = 0, steps = 0, matvecs = 0, nn2s = 0;
};

// Per-kernel-class device timing (CUDA events around each launch on the
// solver's stream), enabled for benchmarks only.
enum KClass { K_SYMV_S = 0, K_SYMV_Q, K_SWEEP, K_SGOP, K_NCLASS };
struct KProf {
  bool on = false;
  double ms[K_NCLASS] = {0};
  long long count[K_NCLASS] = {0};
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<cudaEvent_t> free_;
  cudaEvent_t get() {
    if (free_.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = free_.back();
    free_.pop_back();
    return e;
  }
  void begin(int cls, cudaStream_t st, cudaEvent_t* a) {
    if (!on) return;
    *a = get();
    cudaEventRecord(*a, st);
    pending.push_back({cls, {*a, nullptr}});
  }
  void end(cudaStream_t st) {
    if (!on) return;
    cudaEvent_t b = get();
    cudaEventRecord(b, st);
    pending.back().second.second = b;
  }
  size_t mark() const { return pending.size(); }
  // after the stream has passed the first `upto` pairs (a step that has launched
  // the next step's right-hand side ahead collects only its own)
  void collect(size_t upto = ~size_t(0)) {
    upto = std::min(upto, pending.size());
    for (size_t i = 0; i < upto; ++i) {
      auto& p = pending[i];
      float t = 0;
      if (p.second.second && cudaEventElapsedTime(&t, p.second.first, p.second.second) == cudaSuccess) {
        ms[p.first] += t;
        ++count[p.first];
      }
      free_.push_back(p.second.first);
      if (p.second.second) free_.push_back(p.second.second);
    }
    pending.erase(pending.begin(), pending.begin() + upto);
  }
  void reset() {
    for (int i = 0; i < K_NCLASS; ++i) ms[i] = 0, count[i] = 0;
  }
};

class GpuSolver {
 public:
  explicit GpuSolver(Problem p, std::unique_ptr<Comm> comm = nullptr);
  ~GpuSolver();

  // reference-facing operations (device buffers in/out)
  void apply_block(int op, const double* x, double* y);                 // K11
  void schur_matvec(const double* x, double* y);                        // K1
  // S x without stored S tiles (Problem::implicit_schur): per subdomain
  // A_GG x - A_GI A_II^-1 A_IG x through the local stencils and one interior sweep
  void schur_matvec_implicit(const double* x, double* y);
  // S x over this rank's subdomains (no exchange), optional x.(S x) partial dot
  void s_product(const double* x, double* y, const double* dot_with, double* dot_out);
  void apply_nn2(const double* r, double* z);                           // K2-K4
  // make_preconditioner(schur, kind) (dd.cpp:159-253): 0 nn2, 1 nn1, 2 lumped
  // (nn1 / lumped need Problem::precond == kind: their local operators are
  // built at setup only when selected)
  void apply_precond(int kind, const double* r, double* z);
  int pcg(const double* b, double* x, bool* converged, std::vector<double>* hist);  // K5
  void init_state(const double* u0_nodal_dev, const double* v0_nodal_dev, double f0_scale);
  void set_force_point(int node, double f0, double t0, double amp);
  void set_force_table(const double* table_host, int n_rows);
  // one Newmark step on device; `more`: another step follows in the same call, so
  // its right-hand side may be launched before this step's verdict is read
  int step(int* iters_out, bool more = false);
  std::vector<double> coarse_operator_host() const { return fcc_host_; }
  // dense S_s / S_rr^-1 / Psi_s of local subdomain s (verification hook)
  std::vector<double> local_block(int s, int which, std::vector<long long>* gmap);
  int local_sub(int s_global) const {
    return s_global >= 0 && s_global < G.ns_total ? G.gid_to_local[s_global] : -1;
  }
  void local_dims(int s, long long* d) const { d[0] = NT * ng_[s], d[1] = NT * nr_[s], d[2] = NT * nc_[s]; }
  // full state on every rank (sharded runs: owners' values summed across ranks)
  void gather_state(double* dst_dev);
  int rank() const { return comm_ ? comm_->rank() : 0; }
  int world() const { return comm_ ? comm_->size() : 1; }

  cudaStream_t stream() const { return st_; }
  void set_stream(cudaStream_t s);

  Problem P;
  Geometry G;
  // NG = NT * local interface nodes, NGG = NT * global interface nodes (equal
  // on one GPU), NC = NT * cross points
  int NT = 0, NIN = 0, NS = 0, n = 0, NG = 0, NC = 0;
  long long NGG = 0;
  // C-ABI interface vectors are global; the solver works on the rank's local numbering
  void iface_to_local(const double* glob_dev, double* loc_dev);
  void iface_to_global(const double* loc_dev, double* glob_dev);
  size_t NSTATE = 0;
  double setup_s = 0;
  Timers T;
  KProf KP;
  // device memory this solver allocated during setup (the process-wide count
  // grew by this much while the constructor ran; concurrent constructions
  // in one process blur it)
  long long device_bytes() const { return setup_bytes_; }
  long long setup_bytes_ = 0;
  // algorithmic bytes: unique symmetric entries of all S_s / Q_s
  double bytes_S() const;
  double bytes_Q() const;
  double bytes_sweep() const;  // one forward+backward interior solve
  double bytes_sgop() const;   // one global transient SG-operator apply
  double flops_sgop() const;   // algorithmic flops of that apply
  double bytes_iter() const;   // one PCG iteration (SURVEY 8d B_iter)

  // state
  DBuf<double> u, v, a, um, uc, unext;
  double t_now = 0.0;
  int step_index = 0;
  // probes (device history) filled per step
  std::vector<int> probe_dofs;
  DBuf<int> d_probe_dofs, d_probe_own;  // own: sharded runs, probe dof owned by this rank
  DBuf<double> probe_hist;  // [step][probe][2 + P+1]: mean, std, u_0 .. u_P
  int probe_cap = 0;
  void record_probes(int step, const int* conv = nullptr);  // conv: skip unless *conv (device flag)
  double last_rel = 0.0;  // final true residual of the last PCG solve

 private:
  std::unique_ptr<Comm> comm_;  // null on a single GPU
  void allreduce(double* buf, size_t n) {
    if (comm_) comm_->allreduce_sum(buf, n, st_);
  }
  DBuf<double> own_mask_;  // sharded: 1 on dofs this rank owns (Geometry::owner_of_dof), per term
  // sharded interface halo (host.hpp Halo, tiles.cuh HaloDev; shard.cu)
  DBuf<int> hx_pk_ptr_, hx_cnode_, hx_cptr_;
  DBuf<int2> hx_pk_, hx_csrc_;
  DBuf<double> hx_send_, hx_recv_;
  std::vector<size_t> hx_off_, hx_cnt_;  // per peer block, doubles
  int hx_nshared_ = 0;
  DBuf<double> own_w_;  // NG: 1 on the interface entries this rank owns (dots); sharded only
  DBuf<int> sub_gid_d_, gid_local_d_, iface_gpos_d_;
  void build_halo();
  HaloDev halo_dev() const;
  void halo_exchange();
  void halo_sum(double* y);  // complete a local partial interface vector (no-op unsharded)
  const double* dot_mask() const { return comm_ ? own_w_.p : nullptr; }
  void build_device_inputs(const Stencils& st);
  void setup_interior_and_schur(int b0, int nb);
  void plan_nn2();
  void nn2_batch(int b0, int nb, std::vector<double>& fcc);
  void finish_nn2(std::vector<double>& fcc);
  void build_maps();
  void sweep(double* x);  // x <- A_II^-1 x (block-row layout, all subdomains)
  void gather_li(const double* glob, double* li, bool weighted);
  void scatter_li(const double* li, double* glob, bool weighted, double* dot_with, double* dot_out);
  void symv(TilePack& tp, const double* xloc, double* yloc_or_null);
  double dot_host(const double* a, const double* b, long long len, bool iface);
  void dot_dev(const double* a, const double* b, long long len, double* out, bool iface);
  void local_force(double fext);
  void mass_solve(double* x, const double* b);
  LocalArgs local_args() const;
  const double* force_at(double t, int row, double* fval);

  cudaStream_t st_ = nullptr;
  bool own_stream_ = false;
  cublasHandle_t blas_ = nullptr;
  cusolverDnHandle_t sol_ = nullptr;

  // tensor: lists by output term k (i, j, g) and by pair (k, j) (i, g)
  DBuf<int> gk_ptr, gk_i, gk_j, gp_ptr, gp_i;
  DBuf<double> gk_v, gp_v;
  // stencils
  DBuf<double> Kg, Mg, Kl, Ml;
  // tiled global stencils and the JIT SG operator (sgop.cu)
  DBuf<double> Kp_, Kpart_, yglob_;
  // (s * nl + lid) lists: interface nodes, interior nodes next to the interface
  DBuf<int> ilist_, alist_;
  long long n_ilist_ = 0, n_alist_ = 0;
  SgOpArgs sgop_args_{};  // global-grid operator: stencils, shapes and TMA maps
  std::shared_ptr<SgOpJit> sgop_;
  // geometry maps
  DBuf<int> lid_to_p;           // [s * nl + lid]
  DBuf<int> iface_pos;          // per subdomain local p -> global iface pos, flat with ip_off
  DBuf<double> iface_w;
  DBuf<int> ip_off;             // ns + 1
  DBuf<int> inv_cnt, inv_s, inv_p;  // per global interface node: <= 4 (s, p), ascending s
  DBuf<int> cinv_cnt, cinv_s, cinv_c;  // per corner node: <= 4 (s, local corner index)
  DBuf<int> r_gidx, c_gidx;     // NN2 gather: r-space / c-space -> global flat, per subdomain padded
  DBuf<double> r_w, c_w;
  DBuf<int> iface_of_dof;       // reduced dof -> global interface position or -1
  DBuf<int> pkind_;             // flat (ip_off): remaining index rho >= 0, or -1 - corner index
  DBuf<int> cpos_flat_, cp_off_;  // per subdomain local corner -> global corner position
  DBuf<int> ng_d, nr_d, nc_d;
  std::vector<int> ng_, nr_, nc_;
  std::vector<long long> roff_, coff_, psioff_;
  DBuf<long long> d_roff, d_coff, d_psioff;

  // PCG matrices (Sinvp: S_s^-1 for NN1, Aggp: A_GG,s for lumped; only when selected)
  TilePack Sp, Qp, Sinvp, Aggp;
  void apply_one_level(TilePack& tp, const double* r, double* z);
  DBuf<double> Psi, Finv;
  std::vector<double> fcc_host_;
  // interior factor
  int B = 0, amax_ = 0;
  DBuf<double> Sdense_;  // setup only
  DBuf<int> iface_lid_;  // flat (ip_off): local interface p -> local node id
  DBuf<double> Linv, Lsub;  // dense setup copies (freed after compaction)
  DBuf<double> Fcomp;       // compact interior factor (sweep.cu)
  DBuf<int> sw_off, sw_cuts, sw_ncut, sw_wcuts, sw_nw;
  int sweep_cs_ = 1, sweep_nch_ = 0, sweep_nbm_ = 12;
  bool sweep_generic_ = false;  // large interior blocks: sweep_generic_kernel
  bool sweep_small_ = false;    // small interior blocks (B <= 96): sweep_small_kernel, one warp per subdomain
  bool direct_ = false;          // one subdomain, no interface (sg.cpp:146): the step is one interior solve
  long long sweep_lo_off_ = 0, sweep_up_off_ = 0;
  SweepLayout* sweep_layout_ = nullptr;
  void build_sweep_layout();
  void extract_band_batch(int b0, int nb);
  void compact_dinv_batch(int b0, int nb, const double* dinv);
  size_t sweep_smem_bytes() const;
  // persistent cooperative PCG (pcg_fused.cu)
  void setup_fused_pcg();
  int pcg_fused(const double* b, double* x, bool* converged, std::vector<double>* hist);
  void pcg_fused_launch(const double* b, double* x);
  int pcg_fused_finish(bool* converged, std::vector<double>* hist);
  bool fused_ok() const { return use_fused_ && !comm_ && P.precond == 0 && !P.implicit_schur; }
  bool phase_ok() const { return use_phase_ && walk_ok_ && P.precond == 0 && !P.implicit_schur; }
  // phase-split PCG (pcg_fused.cu): sharded runs, or SGW_PCG=phase on one GPU
  struct FusedPcg fused_args(const double* b, double* x) const;
  void phase_seq(int which, const struct FusedPcg& A);
  bool build_phase_graphs(const double* b, double* x);
  int pcg_phase(const double* b, double* x, bool* converged, std::vector<double>* hist);
  bool use_phase_ = true, ph_graph_ok_ = true;
  DBuf<double> ph_xch_, ph_sc_;
  DBuf<int> ph_st_;
  int* h_st_ = nullptr;
  cudaGraphExec_t ph_graph_[4] = {nullptr, nullptr, nullptr, nullptr};
  long long ph_graph_launches_[4] = {0, 0, 0, 0};
  const double* ph_graph_b_ = nullptr;
  const double* ph_graph_x_ = nullptr;
  double* h_fused_ = nullptr;  // pinned: persistent PCG outputs [4 ints as doubles' room][history]
  DBuf<int> fused_out_;
  RangeBufs rs_, rq_, rp_;
  bool walk_ok_ = false;  // ranges built: the host-driven loop uses walk_kernel
  void walk_pack(int which, const double* x);  // 0: S, 1: Q
  void walk_psi(int pass, const double* x);     // Psi^T tiles: 1 on [0 | f_r], 2 on [B_s u_c | 0]
  struct RangePack psi_pack() const;
  DBuf<int> psi_ncs_;                            // NT nc_s per subdomain
  struct RangePack range_pack(int which) const;
  // Psi_s^T as rectangular tiles for the persistent kernel (pcg_fused.cu)
  DBuf<double> psi_tiles_;
  DBuf<long long> psi_toff_;
  DBuf<int> psi_tbytes_, psi_dnI_, psi_dnJ_;
  std::vector<int> psi_nI_, psi_nJ_;
  void build_psi_tiles();
  int fused_nst_ = 3, fused_maxlen_ = 0;
  size_t fused_smem_ = 0;
  DBuf<double> fused_part_, fused_hist_, li_z_, li_p_, li_xx_, ucl_;
 public:
  DBuf<double> tphase_;  // per-phase ns of the persistent PCG kernel (profiling)
 private:
  int fused_grid_ = 0;
  bool use_fused_ = true;
  int l2_keep_ = 0;  // persistent PCG: tile loads keep L2 residency (small tile sets)
  // per (interface node, sharing-subdomain slot e < 4) descriptors of the PCG
  // glue (local-input writes and partial reductions), so that a node's slots
  // load in parallel instead of through chains of index lookups
  DBuf<int4> d_ifd_, d_sred_, d_zred_, d_pred_;
  DBuf<double> d_ifw_;
  void build_scatter_desc();
  // work vectors
  DBuf<double> li_x, li_y, r_x, r_t, c_f, c_d, dcoarse, ucoarse;
  DBuf<double> vb, vx, vr, vz, vp, vq, vrt;
  DBuf<double> fI, yI, wI, fG;
  DBuf<double> scal;  // device scalars
  DBuf<double> init_w_, mass_w_;  // init_state / mass_solve work vectors (kept across runs)
  // interface <-> interior coupling blocks (step.cu): per edge (interface node q,
  // interior neighbour i) the (P+1)^2 block of the transient operator A(q, i) =
  // A(i, q); CSR by interface-list entry (A_GI) and by interior-list entry (A_IG)
  DBuf<double> cpl_blk_, frc_blk_;  // frc: local-force stiffness blocks of the interface list
  DBuf<int4> cpl_edge_;  // {s, q lid, i lid, dir}
  DBuf<int> cpl_q_cls_, cpl_iptr_, cpl_iedge_, cpl_aptr_, cpl_aedge_;
  bool cpl_built_ = false;
  void build_coupling_blocks();
  DBuf<double> dpart;
  DBuf<unsigned> dcount;
  // forcing
  int force_kind_ = 0, force_node_ = -1, force_dof_ = -1;
  double force_f0_ = 0, force_t0_ = 0, force_amp_ = 0;
  const double* force_tab_ = nullptr;  // caller's table (valid during sgw_run)
  size_t force_len_ = 0;
  DBuf<double> force_row_, fext_;
 public:
  void drop_force_table() {
    if (force_kind_ == 2) force_kind_ = 0, force_tab_ = nullptr, force_len_ = 0;
  }
  DBuf<double> nodal_u0_, nodal_v0_;  // sgw_run / sgw_init_state: nodal initial fields (kept across calls)
 private:
  cudaEvent_t ev_[10];  // [8], [9]: right-hand-side phase of a step launched ahead
  cudaStream_t side_ = nullptr;  // read-back of the persistent PCG's outputs
  bool rhs_ahead_ = false;  // the next step's right-hand side is already on the stream
  int rhs_par_ = 0;         // event pair of the current step's right-hand side (0: ev_[2..3], 1: ev_[8..9])
  void launch_rhs(double t_next, int row_next, cudaEvent_t e0, cudaEvent_t e1);
  // host-driven PCG: pinned residual scalar and the two per-iteration graphs
  double* h_scal_ = nullptr;
  cudaGraphExec_t graph_mv_ = nullptr, graph_pc_ = nullptr;
  const double* graph_x_ = nullptr;
  long long graph_mv_launches_ = 0, graph_pc_launches_ = 0;
};

}  // namespace sgw
