// TEST INFRASTRUCTURE ONLY — see oracle.hpp.  extern "C" surface of the oracle
// for the Python test harness (oracle/oracle.py, ctypes).  Plain pointers and
// sizes; errors are returned as non-zero codes with orc_last_error() text.
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}
struct Handle {
  Mesh mesh;
  Partition part;
  std::unique_ptr<SgSolver> solver;
  SgHistory last;
};
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// Nodal lognormal PCE coefficients (src/experiments.cpp:113-121 input chain).
// out: n_in x n_nodes, term-major.  Returns n_in via *n_in_out.
int orc_lognormal_coeff(int nx, int ny, double sigma, double bx, double by, double g0, int n_vars,
                        int p_in, double* out, int out_cap, int* n_in_out) {
  try {
    const Mesh mesh = build_unit_square_mesh(nx, ny);
    const KleExpansion kle = kle_exponential(sigma, bx, by, n_vars, mesh, g0);
    const CoefficientField f = lognormal_pce(kle, n_vars, p_in);
    *n_in_out = f.n_terms();
    if (out) {
      if (out_cap < f.n_terms() * mesh.n_nodes()) throw std::invalid_argument("buffer too small");
      for (int i = 0; i < f.n_terms(); ++i)
        std::memcpy(out + size_t(i) * mesh.n_nodes(), f.terms[i].data(), sizeof(double) * mesh.n_nodes());
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// KLE 1D roots and 2D eigenvalues (for spectrum checks).
int orc_kle_lambdas(int nx, int ny, double sigma, double bx, double by, int n_modes, double* lambdas) {
  try {
    const Mesh mesh = build_unit_square_mesh(nx, ny);
    const KleExpansion kle = kle_exponential(sigma, bx, by, n_modes, mesh, 0.0);
    for (int m = 0; m < n_modes; ++m) lambdas[m] = kle.modes[m].lambda;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Triple-product tensor entries (i, j, k<=..., value) with j <= k.  quadrature != 0
// uses the Gauss-Hermite cross-check.  Call with ents == nullptr to size.
int orc_triple_products(int n_vars, int p_in, int p_out, int quadrature, int* n_in, int* n_out,
                        int* n_ent, int* ii, int* jj, int* kk, double* vv) {
  try {
    const TripleTensor t = quadrature ? triple_products_quadrature(n_vars, p_in, p_out)
                                      : triple_products(n_vars, p_in, p_out);
    *n_in = t.n_input;
    *n_out = t.n_output;
    int c = 0;
    for (int i = 0; i < t.n_input; ++i)
      for (const auto& e : t.by_input[i]) {
        if (ii) {
          ii[c] = i;
          jj[c] = e.j;
          kk[c] = e.k;
          vv[c] = e.value;
        }
        ++c;
      }
    *n_ent = c;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int orc_nearest_node(int nx, int ny, double x, double y) {
  return nearest_node(build_unit_square_mesh(nx, ny), x, y);
}

// SgSolver ctor (src/sg.cpp:128-176).  coeff: n_in x n_nodes; tensor entries
// with j <= k as produced by triple_products.
int orc_solver_create(int nx, int ny, int px, int py, int n_in, const double* coeff, int n_out,
                      int n_ent, const int* ei, const int* ej, const int* ek, const double* ev,
                      double density, double alpha0, double alpha1, double gamma, double zeta,
                      double dt, double tol, int max_iter, int threads, int precond, void** out) {
  try {
    auto h = std::make_unique<Handle>();
    h->mesh = build_unit_square_mesh(nx, ny);
    h->part = partition_structured(h->mesh, px, py);
    CoefficientField f;
    for (int i = 0; i < n_in; ++i)
      f.terms.emplace_back(coeff + size_t(i) * h->mesh.n_nodes(), coeff + size_t(i + 1) * h->mesh.n_nodes());
    TripleTensor t;
    t.n_input = n_in;
    t.n_output = n_out;
    t.by_input.resize(n_in);
    for (int c = 0; c < n_ent; ++c) {
      if (ei[c] < 0 || ei[c] >= n_in) throw std::invalid_argument("tensor entry input index out of range");
      t.by_input[ei[c]].push_back({ej[c], ek[c], ev[c]});
    }
    NewmarkParams p;
    p.gamma = gamma;
    p.zeta = zeta;
    p.dt = dt;
    SgOptions o;
    o.tol = tol;
    o.max_iter = max_iter;
    o.threads = threads;
    if (precond < 0 || precond > 2) throw std::invalid_argument("unknown preconditioner");
    o.precond = precond;
    h->solver = std::make_unique<SgSolver>(h->mesh, h->part, f, t, density, alpha0, alpha1, p, o);
    *out = h.release();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void orc_solver_destroy(void* h) { delete static_cast<Handle*>(h); }

// sizes[0..5] = n_dofs, n_terms, n_iface, n_corner, n_global(flat), uses_direct
void orc_solver_sizes(void* hp, long long* sizes) {
  const Handle* h = static_cast<Handle*>(hp);
  const SgSolver& s = *h->solver;
  sizes[0] = s.reduction().n_dofs();
  sizes[1] = s.n_terms();
  sizes[2] = s.layout().n_iface();
  sizes[3] = s.layout().n_corner();
  sizes[4] = s.schur().n_global;
  sizes[5] = s.uses_direct() ? 1 : 0;
}

// op: 0 mass, 1 stiffness, 2 transient (src/sg.cpp:425-447)
int orc_apply_block(void* hp, int op, const double* x, double* y) {
  try {
    const SgSolver& s = *static_cast<Handle*>(hp)->solver;
    const size_t N = size_t(s.n_terms()) * s.reduction().n_dofs();
    const Vec xv(x, x + N);
    const Vec out = op == 0 ? s.apply_block_mass(xv) : op == 1 ? s.apply_block_stiffness(xv) : s.apply_block_transient(xv);
    std::memcpy(y, out.data(), sizeof(double) * N);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// which: 0 matvec (src/dd.cpp:142-157), 1 apply_nn2 (src/dd.cpp:199-253),
//        2 apply_nn1 (:178-195), 3 apply_lumped (:159-176)
int orc_schur_apply(void* hp, int which, const double* x, double* y) {
  try {
    const SgSolver& s = *static_cast<Handle*>(hp)->solver;
    const Vec xv(x, x + s.schur().n_global);
    const Vec out = which == 0   ? s.schur().matvec(xv)
                    : which == 1 ? s.schur().apply_nn2(xv)
                    : which == 2 ? s.schur().apply_nn1(xv)
                                 : s.schur().apply_lumped(xv);
    std::memcpy(y, out.data(), sizeof(double) * out.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int orc_coarse_operator(void* hp, double* out) {
  const SgSolver& s = *static_cast<Handle*>(hp)->solver;
  const Dense& f = s.schur().coarse_operator();
  std::memcpy(out, f.a.data(), sizeof(double) * f.a.size());
  return 0;
}

// pcg(matvec, apply_nn2 / make_preconditioner, rhs, tol, max_iter) on the
// solver's Schur system (src/pcg.cpp:7-50); hist: >= max_iter + 2 entries.
int orc_pcg(void* hp, const double* rhs, double* x, int* iters, int* converged, double* hist, int hist_cap,
            int precond, double tol, int max_iter) {
  try {
    const SgSolver& s = *static_cast<Handle*>(hp)->solver;
    const SchurSystem& sys = s.schur();
    const Vec b(rhs, rhs + sys.n_global);
    PcgReport rep;
    const Vec xv = pcg([&](const Vec& v) { return sys.matvec(v); }, [&](const Vec& v) { return sys.apply(precond, v); },
                       b, tol, max_iter, &rep);
    std::memcpy(x, xv.data(), sizeof(double) * xv.size());
    *iters = rep.iterations;
    *converged = rep.converged ? 1 : 0;
    for (int i = 0; i < hist_cap; ++i) hist[i] = i < int(rep.residual_history.size()) ? rep.residual_history[i] : -1.0;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Local Schur S_s (column-major a x a) and its flat gmap.
int orc_local_schur(void* hp, int s, double* S, long long* gmap, long long* a_out) {
  const SgSolver& sv = *static_cast<Handle*>(hp)->solver;
  const LocalSchur& ls = sv.schur().locals.at(s);
  *a_out = ls.n_flat();
  if (S) std::memcpy(S, ls.S.a.data(), sizeof(double) * ls.S.a.size());
  if (gmap)
    for (Index k = 0; k < ls.n_flat(); ++k) gmap[k] = ls.gmap[k];
  return 0;
}

// the rest of LocalSchur s (dd.hpp:50-62): weights, r_idx, c_idx, corner_gmap
// (NULL pointers: sizes only)
int orc_local_maps(void* hp, int s, double* w, int* r_idx, int* c_idx, long long* corner_gmap, long long* nr,
                   long long* nc) {
  const SgSolver& sv = *static_cast<Handle*>(hp)->solver;
  const LocalSchur& ls = sv.schur().locals.at(s);
  *nr = (long long)ls.r_idx.size(), *nc = (long long)ls.c_idx.size();
  if (w)
    for (Index k = 0; k < ls.n_flat(); ++k) w[k] = ls.weights[k];
  if (r_idx)
    for (size_t k = 0; k < ls.r_idx.size(); ++k) r_idx[k] = int(ls.r_idx[k]);
  if (c_idx)
    for (size_t k = 0; k < ls.c_idx.size(); ++k) c_idx[k] = int(ls.c_idx[k]);
  if (corner_gmap)
    for (size_t k = 0; k < ls.corner_gmap.size(); ++k) corner_gmap[k] = ls.corner_gmap[k];
  return 0;
}

// SgSolver::run (src/sg.cpp:358-423).  Force: Ricker wavelet
//   amp * (1 - 2 pi^2 f0^2 (t - t0)^2) exp(-pi^2 f0^2 (t - t0)^2)
// at mesh node force_node (force_node < 0: no forcing).  Outputs: iters[n_steps],
// final true residual per step res[n_steps]; full (optional) (n_steps+1) x N.
int orc_run(void* hp, const double* u0, const double* v0, int n_steps, int force_node, double f0,
            double t0, double amp, int* iters, double* res, double* full, int n_probes,
            const int* probe_nodes, double* probe_mean, double* probe_std) {
  try {
    Handle* h = static_cast<Handle*>(hp);
    SgSolver& s = *h->solver;
    const Index nn = h->mesh.n_nodes();
    ForceFn force;
    if (force_node >= 0) {
      force = [=](double t) {
        Vec f(nn, 0.0);
        const double a = M_PI * M_PI * f0 * f0 * (t - t0) * (t - t0);
        f[force_node] = amp * (1.0 - 2.0 * a) * std::exp(-a);
        return f;
      };
    }
    s.set_store_full(full != nullptr);
    s.set_probes(std::vector<Index>(probe_nodes, probe_nodes + n_probes));
    SgHistory hist = s.run(Vec(u0, u0 + nn), Vec(v0, v0 + nn), n_steps, force);
    for (int p = 0; p < n_probes; ++p)
      for (int k = 0; k <= n_steps; ++k) {
        probe_mean[size_t(p) * (n_steps + 1) + k] = hist.probe_mean[p][k];
        probe_std[size_t(p) * (n_steps + 1) + k] = hist.probe_std[p][k];
      }
    for (size_t k = 0; k < hist.reports.size(); ++k) {
      if (iters) iters[k] = hist.reports[k].iterations;
      if (res) res[k] = hist.reports[k].residual_history.back();
    }
    if (full) {
      const size_t N = size_t(s.n_terms()) * s.reduction().n_dofs();
      for (size_t k = 0; k < hist.full_state.size(); ++k)
        std::memcpy(full + k * N, hist.full_state[k].data(), sizeof(double) * N);
    }
    h->last = std::move(hist);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// residual history of step k of the last run; returns its length
int orc_residual_history(void* hp, int k, double* out, int cap) {
  const Handle* h = static_cast<Handle*>(hp);
  const auto& rh = h->last.reports.at(k).residual_history;
  for (int i = 0; i < int(rh.size()) && i < cap; ++i) out[i] = rh[i];
  return int(rh.size());
}

// test_dd.cpp:123-151: one LocalSchur with S = a (column-major n x n), identity
// gmap, unit weights, no corners.  Returns z = NN2(r) and the PCG iteration count.
int orc_single_block_nn2(int n, const double* a, const double* r, double* z, double tol, int* iters) {
  try {
    SchurSystem sys;
    LocalSchur ls;
    ls.S = Dense(n, n);
    std::memcpy(ls.S.a.data(), a, sizeof(double) * n * n);
    ls.weights.assign(n, 1.0);
    for (int i = 0; i < n; ++i) {
      ls.gmap.push_back(i);
      ls.r_idx.push_back(i);
    }
    sys.n_global = n;
    sys.n_corner = 0;
    sys.locals.push_back(std::move(ls));
    sys.finalize(false);
    const Vec rv(r, r + n);
    const Vec zv = sys.apply_nn2(rv);
    std::memcpy(z, zv.data(), sizeof(double) * n);
    PcgReport rep;
    pcg([&](const Vec& v) { return sys.matvec(v); }, [&](const Vec& v) { return sys.apply_nn2(v); }, rv, tol,
        50, &rep);
    *iters = rep.converged ? rep.iterations : -1;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// One subdomain's local operators without building the whole solver
// (SgSolver::local_blocks): for checking the GPU tiles at sizes where the full
// oracle does not fit in host memory.  sizes_out = {a, r, c}.
int orc_local_blocks_create(int nx, int ny, int px, int py, int n_in, const double* coeff, int n_out, int n_ent,
                            const int* ei, const int* ej, const int* ek, const double* ev, double density,
                            double alpha0, double alpha1, double gamma, double zeta, double dt, int s, int threads,
                            long long* sizes_out, void** out) {
  try {
    const Mesh mesh = build_unit_square_mesh(nx, ny);
    const Partition part = partition_structured(mesh, px, py);
    CoefficientField f;
    for (int i = 0; i < n_in; ++i)
      f.terms.emplace_back(coeff + size_t(i) * mesh.n_nodes(), coeff + size_t(i + 1) * mesh.n_nodes());
    TripleTensor t;
    t.n_input = n_in;
    t.n_output = n_out;
    t.by_input.resize(n_in);
    for (int c = 0; c < n_ent; ++c) t.by_input.at(ei[c]).push_back({ej[c], ek[c], ev[c]});
    NewmarkParams p;
    p.gamma = gamma, p.zeta = zeta, p.dt = dt;
    auto ls = std::make_unique<LocalSchur>(SgSolver::local_blocks(mesh, part, f, t, density, alpha0, alpha1, p, s,
                                                                  threads));
    sizes_out[0] = ls->n_flat();
    sizes_out[1] = Index(ls->r_idx.size());
    sizes_out[2] = Index(ls->c_idx.size());
    *out = ls.release();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// S (a x a column-major) and gmap (a); qv = S_rr^{-1} v for m vectors v
// (r x m column-major); psi = S_rr^{-1} S_rc (r x c column-major).  Any
// output may be null.
int orc_local_blocks_get(void* hp, double* S, long long* gmap, const double* v, int m, double* qv, double* psi) {
  try {
    const LocalSchur& ls = *static_cast<LocalSchur*>(hp);
    const Index r = Index(ls.r_idx.size()), c = Index(ls.c_idx.size());
    if (S) std::memcpy(S, ls.S.a.data(), sizeof(double) * ls.S.a.size());
    if (gmap)
      for (Index k = 0; k < ls.n_flat(); ++k) gmap[k] = ls.gmap[k];
    if (qv)
      for (int q = 0; q < m; ++q) {
        std::memcpy(qv + size_t(q) * r, v + size_t(q) * r, sizeof(double) * r);
        ls.Srr_llt.solve_in_place(qv + size_t(q) * r);
      }
    if (psi)
      parallel_for(c, 8, [&](int b) {
        double* col = psi + size_t(b) * r;
        for (Index a = 0; a < r; ++a) col[a] = ls.S_rc(a, b);
        ls.Srr_llt.solve_in_place(col);
      });
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void orc_local_blocks_destroy(void* hp) { delete static_cast<LocalSchur*>(hp); }

void orc_timing(void* hp, double* out) {
  const SgSolver& s = *static_cast<Handle*>(hp)->solver;
  out[0] = s.t_setup;
  out[1] = s.t_pcg;
  out[2] = s.t_steps;
  out[3] = double(s.total_iterations);
}

}  // extern "C"
