// =============================================================================
// TEST INFRASTRUCTURE ONLY — CPU oracle for the SG-PCG / NN2 hot path.
//
// A plain C++17 restatement (no Eigen, no BLAS) of the reference `sgwave`
// algorithm for the per-Newmark-step interface-Schur PCG solve preconditioned
// by the two-level Neumann-Neumann (NN2) domain decomposition.  It exists so
// that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg have an
// independent checker.  It is NEVER linked into, imported by or called from
// the product library (paper_2512_23027_b200/).
//
// Every function cites the reference file:line it restates (paths relative to
// the reference's proj/ directory).  Divergences from the reference, all
// rounding-level or documented in DESIGN.md:
//   * triple_products: the `order_in <= order_out` guard (src/pce.cpp:97-99)
//     is lifted — the BASELINE configs use p_in = 2 p_out.
//   * The interior Dirichlet factor uses a node-major banded Cholesky instead
//     of Eigen's SimplicialLLT+AMD (src/sg.cpp:218-225); same matrix, same
//     maths, different elimination order (differences ~1e-15 relative).
//   * Dense kernels (GEMV/Cholesky) sum in their own order.
// Parity pins: see tests/test_oracle.py (reference test properties and the
// recorded iteration counts of proj/test_output.txt:44 and :52).
// =============================================================================
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace oracle {

using Index = int;
using Vec = std::vector<double>;

// ---------------------------------------------------------------- mesh ------
// include/sgwave/mesh.hpp:13-24, src/mesh.cpp:15-58
struct Mesh {
  int nx = 0, ny = 0;
  std::vector<double> x, y;                  // node coordinates
  std::vector<std::array<int, 3>> elements;  // CCW triangles
  std::vector<Index> dirichlet_nodes;        // sorted
  double h = 0.0;
  Index n_nodes() const { return static_cast<Index>(x.size()); }
  Index n_elements() const { return static_cast<Index>(elements.size()); }
};
Mesh build_unit_square_mesh(int nx, int ny);
Index nearest_node(const Mesh& mesh, double x, double y);  // src/mesh.cpp:83-96

// ----------------------------------------------------------- partition ------
// include/sgwave/partition.hpp:25-43, src/partition.cpp:48-133
struct Partition {
  int n_sub = 0;
  std::vector<std::vector<Index>> subdomain_elements, subdomain_nodes, interior_nodes,
      interface_nodes;
  std::vector<Index> global_interface, corner_nodes, remaining_nodes;
  std::vector<int> multiplicity;
  int multiplicity_of(Index node) const;
};
Partition partition_structured(const Mesh& mesh, int px, int py);

// --------------------------------------------------------- reduction --------
// src/assembly.cpp:121-158
struct DirichletReduction {
  std::vector<Index> node_to_dof, dof_to_node;
  Index n_dofs() const { return static_cast<Index>(dof_to_node.size()); }
  Vec reduce_vector(const Vec& nodal) const;
};
DirichletReduction make_dirichlet_reduction(const Mesh& mesh);

// ------------------------------------------------------ sparse (CSR) --------
// Triplets are summed in insertion order, like Eigen's setFromTriplets.
struct Triplet {
  Index r, c;
  double v;
};
struct Csr {
  Index rows = 0, cols = 0;
  std::vector<Index> ptr, col;
  std::vector<double> val;
  static Csr from_triplets(Index rows, Index cols, std::vector<Triplet> trips);
  void apply(const double* x, double* y, double alpha = 1.0, bool accumulate = false) const;
  void apply_t(const double* x, double* y) const;  // y += A^T x
  double at(Index r, Index c) const;
};
Csr assemble_stiffness_reduced(const Mesh& mesh, const Vec& coeff, const DirichletReduction& red);
Csr assemble_mass_reduced(const Mesh& mesh, double density, const DirichletReduction& red);

// ---------------------------------------------------------- stochastic ------
// src/pce.cpp:19-37, :60-67, :96-122 ; src/kle.cpp ; src/lognormal.cpp
std::vector<std::vector<int>> multi_indices(int n_vars, int max_order);
double hermite(int n, double x);
struct TripleTensor {
  struct Entry {
    int j, k;
    double value;
  };
  int n_input = 0, n_output = 0;
  std::vector<std::vector<Entry>> by_input;  // j <= k only
  template <typename F>
  void for_each(int i, F&& f) const {
    for (const Entry& e : by_input[i]) {
      f(e.j, e.k, e.value);
      if (e.j != e.k) f(e.k, e.j, e.value);
    }
  }
};
TripleTensor triple_products(int n_vars, int order_in, int order_out);
TripleTensor triple_products_quadrature(int n_vars, int order_in, int order_out);

struct KleMode {
  double lambda = 0.0;
  Vec phi;
};
struct Kle1dMode {
  double omega = 0.0, lambda = 0.0;
  bool even = true;
};
std::vector<Kle1dMode> kle_eigens_1d(double b, int n_modes);
double kle_eigenfunction_1d(const Kle1dMode& m, double x);
struct KleExpansion {
  double sigma = 0.0, bx = 1.0, by = 1.0, mean = 0.0;
  std::vector<KleMode> modes;
};
KleExpansion kle_exponential(double sigma, double bx, double by, int n_modes, const Mesh& mesh,
                             double mean);
struct CoefficientField {
  std::vector<Vec> terms;
  int n_terms() const { return static_cast<int>(terms.size()); }
};
CoefficientField lognormal_pce(const KleExpansion& kle, int n_vars, int p_in);

// --------------------------------------------------------------- dense ------
// column-major dense matrix (Eigen's default layout)
struct Dense {
  Index rows = 0, cols = 0;
  std::vector<double> a;
  Dense() = default;
  Dense(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
  double& operator()(Index r, Index c) { return a[static_cast<size_t>(c) * rows + r]; }
  double operator()(Index r, Index c) const { return a[static_cast<size_t>(c) * rows + r]; }
};
// Lower Cholesky factor with Eigen's LLT failure semantics (pivot <= 0).
struct Llt {
  Index n = 0;
  std::vector<double> l;  // row-major lower: l[i*n + j], j <= i
  bool ok = false;
  bool compute(const Dense& m);
  void solve_in_place(double* b) const;  // b <- M^{-1} b
};
Llt llt_regularized(Dense m);  // src/dd.cpp:66-76

// Node-major banded Cholesky of an SPD matrix given in its own index space.
struct BandLlt {
  Index n = 0, bw = 0;
  std::vector<double> l;  // row band: l[i*(bw+1) + (j - i + bw)], i-bw <= j <= i
  bool compute(Index n, Index bw, const std::function<void(Index, double*)>& fill_row);
  void solve_in_place(double* b) const;
  void solve_many(double* b, Index nrhs) const;  // b row-major n x nrhs
};

// ------------------------------------------------------------------ dd ------
// include/sgwave/dd.hpp:17-62, src/dd.cpp:10-96
struct SubdomainDofs {
  std::vector<Index> interior, iface, iface_pos, r_local, c_local, corner_pos, loc_dofs;
  Vec weights;
  Index n_interior() const { return static_cast<Index>(interior.size()); }
  Index n_iface() const { return static_cast<Index>(iface.size()); }
};
struct InterfaceLayout {
  std::vector<Index> iface_dofs, corner_dofs;
  std::vector<SubdomainDofs> sub;
  Index n_iface() const { return static_cast<Index>(iface_dofs.size()); }
  Index n_corner() const { return static_cast<Index>(corner_dofs.size()); }
};
InterfaceLayout build_interface_layout(const Partition& part, const DirichletReduction& red);

struct LocalSchur {
  Dense S;
  Dense Kgg;  // flattened interface block A_GG (lumped preconditioner's gg_action, det_loop.cpp:165-167)
  Llt S_llt;  // llt_regularized(S) (NN1, dd.cpp:115)
  std::vector<Index> gmap, r_idx, c_idx, corner_gmap;
  Vec weights;
  Dense S_rc;
  Llt Srr_llt;
  Index n_flat() const { return static_cast<Index>(gmap.size()); }
};
LocalSchur make_flat_maps(const SubdomainDofs& sd, int n_blocks, Index n_iface, Index n_corner);

class SchurSystem {  // include/sgwave/dd.hpp:71-96
 public:
  Index n_global = 0, n_corner = 0;
  int n_threads = 1;
  std::vector<LocalSchur> locals;
  void finalize(bool build_nn1);       // src/dd.cpp:98-140
  Vec matvec(const Vec& x) const;      // src/dd.cpp:142-157
  Vec apply_lumped(const Vec& r) const;  // src/dd.cpp:159-176 (gg_action = Kgg)
  Vec apply_nn1(const Vec& r) const;   // src/dd.cpp:178-195
  Vec apply_nn2(const Vec& r) const;   // src/dd.cpp:199-253
  Vec apply(int kind, const Vec& r) const;  // make_preconditioner: 0 nn2, 1 nn1, 2 lumped
  const Dense& coarse_operator() const { return fcc_; }

 private:
  Dense fcc_;
  Llt fcc_llt_;
  bool has_coarse_ = false;
};

// ----------------------------------------------------------------- pcg ------
// include/sgwave/pcg.hpp:9-21, src/pcg.cpp:7-50
struct PcgReport {
  int iterations = 0;
  bool converged = false;
  std::vector<double> residual_history;
};
using LinearOp = std::function<Vec(const Vec&)>;
Vec pcg(const LinearOp& op, const LinearOp& precond, const Vec& rhs, double tol, int max_iter,
        PcgReport* report);

// ------------------------------------------------------------------ sg ------
struct NewmarkParams {  // include/sgwave/newmark.hpp:11-19
  double gamma = 0.5, zeta = 0.25, dt = 0.0;
  double mass_factor() const { return 1.0 / (zeta * dt * dt); }
  double damping_factor() const { return gamma / (zeta * dt); }
};
struct SgOptions {  // include/sgwave/sg.hpp:15-21 (+ SolveOptions::precond, det_loop.hpp:14)
  int precond = 0;  // 0 nn2 (the SG path, sg.cpp:330), 1 nn1, 2 lumped
  double tol = 1e-8;
  int max_iter = 500;
  int threads = 1;
  bool store_full = false;
  std::vector<Index> probe_nodes;
};
struct SgHistory {
  std::vector<double> times;
  std::vector<std::vector<double>> probe_mean, probe_std;  // [probe][step]
  std::vector<Vec> full_state;
  std::vector<PcgReport> reports;
  double mean_iterations() const;
};
using ForceFn = std::function<Vec(double)>;  // nodal force over all mesh nodes

class SgSolver {  // include/sgwave/sg.hpp:43-98
 public:
  SgSolver(const Mesh& mesh, const Partition& part, const CoefficientField& coeff,
           const TripleTensor& tensor, double density, double alpha0, double alpha1,
           NewmarkParams params, SgOptions options);
  SgHistory run(const Vec& u0_nodal, const Vec& v0_nodal, int n_steps, const ForceFn& force);
  int n_terms() const { return n_terms_; }
  const DirichletReduction& reduction() const { return red_; }
  const InterfaceLayout& layout() const { return layout_; }
  const SchurSystem& schur() const { return schur_; }
  bool uses_direct() const { return direct_; }
  void set_store_full(bool v) { opt_.store_full = v; }
  void set_probes(std::vector<Index> nodes) { opt_.probe_nodes = std::move(nodes); }
  double mass_scale() const { return mass_scale_; }
  double stiff_scale() const { return stiff_scale_; }
  Vec apply_block_mass(const Vec& flat) const;
  Vec apply_block_stiffness(const Vec& flat) const;
  Vec apply_block_transient(const Vec& flat) const;
  static LocalSchur local_blocks(const Mesh& mesh, const Partition& part, const CoefficientField& coeff,
                                 const TripleTensor& tensor, double density, double alpha0, double alpha1,
                                 NewmarkParams params, int s, int threads);

  // per-phase timing of the last run (seconds)
  double t_setup = 0.0, t_pcg = 0.0, t_steps = 0.0;
  long long total_iterations = 0;

  struct StateTriple {
    Vec u, v, a;
    double t = 0.0;
  };

 private:
  struct Local {
    Csr mass;
    std::vector<Csr> k_terms;
    Csr a_ig;  // flattened term-major interior x interface block
    BandLlt ii;
    std::vector<Index> perm;  // term-major flat interior index -> band index
    bool has_interior = false;
  };
  struct Ctx {
    const Mesh& mesh;
    const Partition& part;
    const DirichletReduction& red;
    const InterfaceLayout& layout;
    const CoefficientField& coeff;
    const TripleTensor& tensor;
    double density, mass_scale, stiff_scale;
    int nt, precond;
  };
  static void build_local(const Ctx& cx, int s, int panel_threads, Local& loc, LocalSchur& ls);
  void assemble_subdomains();
  Vec local_force(int s, const Vec& um, const Vec& uc, const Vec& f_next) const;
  Vec step_rhs_and_solve(const StateTriple& st, const Vec& f_next, PcgReport* rep);
  void interior_solve(int s, double* flat) const;  // flat term-major interior vector

  Mesh mesh_;
  Partition part_;
  DirichletReduction red_;
  InterfaceLayout layout_;
  CoefficientField coeff_;
  TripleTensor tensor_;
  int n_terms_;
  double density_, alpha0_, alpha1_;
  NewmarkParams params_;
  SgOptions opt_;
  bool direct_ = false;
  double mass_scale_ = 0.0, stiff_scale_ = 0.0;
  std::vector<Csr> k_red_;
  Csr mass_red_;
  BandLlt mass_llt_, direct_llt_;
  Index direct_bw_ = 0;
  std::vector<Local> locals_;
  SchurSystem schur_;
};

// parallel_for with per-index slots (include/sgwave/parallel.hpp:20-43)
void parallel_for(int n, int n_threads, const std::function<void(int)>& fn);

}  // namespace oracle
