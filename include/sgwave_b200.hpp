// C++ host-side mirror of the reference solver interface for the hot path,
// header-only over the C ABI (include/sgw.h).  Names, argument meaning and
// error behaviour follow the reference:
//   NewmarkParams                 proj/include/sgwave/newmark.hpp:11-19
//   SgOptions, SgHistory          proj/include/sgwave/sg.hpp:13-31
//   SgSolver(ctor, run, apply_block_*, schur, n_terms, uses_direct)   sg.hpp:43-98
//   SchurSystem::matvec / apply_nn2 / coarse_operator                 dd.hpp:71-96
//   PcgReport, pcg(matvec, precond, rhs, tol, max_iter)               pcg.hpp:11-21
// Eigen vectors become std::vector<double>; the mesh and the partition are
// given by their structured sizes (build_unit_square_mesh(nx, ny),
// partition_structured(mesh, px, py)).  Invalid arguments throw
// std::invalid_argument, factorization / convergence / CUDA failures
// std::runtime_error, as the reference does.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sgw.h"

namespace sgwave::b200 {

using Vec = std::vector<double>;
using ForceFn = std::function<Vec(double)>;  // nodal load at time t (det_loop.hpp:32)

struct NewmarkParams {  // newmark.hpp:11-19
  double gamma = 0.5;
  double zeta = 0.25;
  double dt = 0.0;
};

enum class PrecondKind { lumped, nn1, nn2 };  // dd.hpp:98
inline int precond_code(PrecondKind k) { return k == PrecondKind::nn2 ? 0 : k == PrecondKind::nn1 ? 1 : 2; }
inline PrecondKind precond_from_string(const std::string& name) {  // dd.hpp:100
  if (name == "lumped") return PrecondKind::lumped;
  if (name == "nn1") return PrecondKind::nn1;
  if (name == "nn2") return PrecondKind::nn2;
  throw std::invalid_argument("unknown preconditioner: " + name);
}

struct SgOptions {  // sg.hpp:13-19 (threads: accepted, unused on the GPU) + SolveOptions::precond
  PrecondKind precond = PrecondKind::nn2;
  bool implicit_schur = false;  // reduced-memory mode (include/sgw.h)
  double tol = 1e-8;
  int max_iter = 500;
  int threads = 1;
  bool store_full = false;
  std::vector<int> probe_nodes;
  int device = 0;
};

struct PcgReport {  // pcg.hpp:11-18
  int iterations = 0;
  bool converged = false;
  std::vector<double> residual_history;
};

struct SgHistory {  // sg.hpp:21-31
  std::vector<double> times;
  std::vector<Vec> probe_mean, probe_std;  // [probe][step]
  std::vector<std::vector<Vec>> probe_coeffs;  // [probe][term][step]
  std::vector<Vec> full_state;             // [step] flattened (P+1) n_dofs, if requested
  std::vector<PcgReport> reports;
  double mean_iterations() const {
    if (reports.empty()) return 0.0;
    double s = 0.0;
    for (const auto& r : reports) s += r.iterations;
    return s / double(reports.size());
  }
};

struct StructuredMesh {  // build_unit_square_mesh(nx, ny)
  int nx = 0, ny = 0;
  int n_nodes() const { return (nx + 1) * (ny + 1); }
};
struct StructuredPartition {  // partition_structured(mesh, px, py)
  int px = 1, py = 1;
};
struct CoefficientField {  // lognormal_pce(...): terms[i] = nodal values of input term i
  std::vector<Vec> terms;
};
struct TripleEntry {
  int j, k;
  double value;
};
struct TripleTensor {  // pce.hpp:24-40: entries with j <= k, grouped by input term
  int n_input = 0, n_output = 0;
  std::vector<std::vector<TripleEntry>> by_input;
};

namespace detail {
inline void check(int rc) {
  if (rc == SGW_OK) return;
  if (rc == SGW_EINVAL) throw std::invalid_argument(sgw_last_error());
  throw std::runtime_error(sgw_last_error());
}
}  // namespace detail

// Input builders of the reference (kle.cpp / lognormal.cpp / pce.cpp)
inline CoefficientField lognormal_coeff(int nx, int ny, double sigma, double bx, double by, int n_vars, int p_in,
                                        double g0 = 0.0) {
  int n_in = 0;
  detail::check(sgw_lognormal_coeff(nx, ny, sigma, bx, by, g0, n_vars, p_in, nullptr, 0, &n_in));
  const size_t nn = size_t(nx + 1) * (ny + 1);
  Vec flat(size_t(n_in) * nn);
  detail::check(sgw_lognormal_coeff(nx, ny, sigma, bx, by, g0, n_vars, p_in, flat.data(), (long long)flat.size(), &n_in));
  CoefficientField f;
  for (int i = 0; i < n_in; ++i) f.terms.emplace_back(flat.begin() + i * nn, flat.begin() + (i + 1) * nn);
  return f;
}
inline TripleTensor triple_products(int n_vars, int p_in, int p_out) {
  int ni = 0, no = 0, ne = 0;
  detail::check(sgw_triple_products(n_vars, p_in, p_out, &ni, &no, &ne, nullptr, nullptr, nullptr, nullptr, 0));
  std::vector<int> ei(ne), ej(ne), ek(ne);
  Vec ev(ne);
  detail::check(sgw_triple_products(n_vars, p_in, p_out, &ni, &no, &ne, ei.data(), ej.data(), ek.data(), ev.data(), ne));
  TripleTensor t;
  t.n_input = ni, t.n_output = no;
  t.by_input.resize(ni);
  for (int e = 0; e < ne; ++e) t.by_input[ei[e]].push_back({ej[e], ek[e], ev[e]});
  return t;
}
inline int nearest_node(const StructuredMesh& m, double x, double y) { return sgw_nearest_node(m.nx, m.ny, x, y); }

class SgSolver;

class SchurSystem {  // dd.hpp:71-96 (view on the solver's interface system)
 public:
  explicit SchurSystem(sgw_solver* h, long long n_global, long long n_coarse)
      : h_(h), n_(n_global), nc_(n_coarse) {}
  long long n_global() const { return n_; }
  Vec matvec(const Vec& x) const {
    Vec y(n_);
    detail::check(sgw_schur_matvec(h_, x.data(), y.data()));
    return y;
  }
  Vec apply_nn2(const Vec& r) const {
    Vec z(n_);
    detail::check(sgw_apply_nn2(h_, r.data(), z.data()));
    return z;
  }
  // make_preconditioner(system, kind)(r) (dd.cpp:159-253); nn1 / lumped need
  // the solver to be built with that preconditioner
  Vec apply_precond(PrecondKind kind, const Vec& r) const {
    Vec z(n_);
    detail::check(sgw_apply_precond(h_, precond_code(kind), r.data(), z.data()));
    return z;
  }
  Vec apply_nn1(const Vec& r) const { return apply_precond(PrecondKind::nn1, r); }
  Vec apply_lumped(const Vec& r) const { return apply_precond(PrecondKind::lumped, r); }
  Vec coarse_operator() const {  // column-major n_coarse x n_coarse
    Vec f(size_t(nc_) * nc_);
    detail::check(sgw_coarse_operator(h_, f.data()));
    return f;
  }
  // pcg(matvec, apply_nn2, rhs, tol, max_iter) on this system (pcg.hpp:20-21)
  std::pair<Vec, PcgReport> pcg(const Vec& rhs, int max_iter) const {
    Vec x(n_);
    int it = 0, conv = 0;
    Vec hist(size_t(max_iter) + 2);
    detail::check(sgw_pcg(h_, rhs.data(), x.data(), &it, &conv, hist.data(), (int)hist.size()));
    PcgReport rep;
    rep.iterations = it, rep.converged = conv != 0;
    for (double v : hist)
      if (v >= 0.0) rep.residual_history.push_back(v);
    return {x, rep};
  }

 private:
  sgw_solver* h_;
  long long n_, nc_;
};

class SgSolver {  // sg.hpp:43-98
 public:
  SgSolver(const StructuredMesh& mesh, const StructuredPartition& part, const CoefficientField& coeff,
           const TripleTensor& tensor, double density, double alpha0, double alpha1, NewmarkParams params,
           SgOptions options)
      : mesh_(mesh), params_(params), opt_(std::move(options)) {
    const size_t nn = size_t(mesh.n_nodes());
    for (const auto& t : coeff.terms)
      if (t.size() != nn) throw std::invalid_argument("SgSolver: coefficient term size does not match the mesh");
    Vec c;
    for (const auto& t : coeff.terms) c.insert(c.end(), t.begin(), t.end());
    std::vector<int> ei, ej, ek;
    Vec ev;
    for (int i = 0; i < (int)tensor.by_input.size(); ++i)
      for (const auto& e : tensor.by_input[i]) ei.push_back(i), ej.push_back(e.j), ek.push_back(e.k), ev.push_back(e.value);
    sgw_problem pr{};
    pr.nx = mesh.nx, pr.ny = mesh.ny, pr.px = part.px, pr.py = part.py;
    pr.n_input = (int)coeff.terms.size(), pr.coeff = c.data();
    pr.n_output = tensor.n_output, pr.n_entries = (int)ev.size();
    pr.ent_i = ei.data(), pr.ent_j = ej.data(), pr.ent_k = ek.data(), pr.ent_v = ev.data();
    pr.density = density, pr.alpha0 = alpha0, pr.alpha1 = alpha1;
    pr.gamma = params.gamma, pr.zeta = params.zeta, pr.dt = params.dt;
    pr.tol = opt_.tol, pr.max_iter = opt_.max_iter, pr.device = opt_.device;
    pr.rank = 0, pr.world_size = 1, pr.nccl_id = nullptr, pr.precond = precond_code(opt_.precond);
    pr.implicit_schur = opt_.implicit_schur ? 1 : 0;
    if (pr.n_input != tensor.n_input)
      throw std::invalid_argument("SgSolver: coefficient terms do not match tensor input size");
    detail::check(sgw_create(&pr, &h_));
    long long s[8];
    detail::check(sgw_sizes(h_, s));
    n_dofs_ = s[0], n_terms_ = (int)s[1], n_global_ = s[4], n_coarse_ = s[1] * s[3];
  }
  ~SgSolver() {
    if (h_) sgw_destroy(h_);
  }
  SgSolver(const SgSolver&) = delete;
  SgSolver& operator=(const SgSolver&) = delete;

  int n_terms() const { return n_terms_; }
  long long n_dofs() const { return n_dofs_; }
  bool uses_direct() const { return false; }
  SchurSystem schur() const { return SchurSystem(h_, n_global_, n_coarse_); }

  Vec apply_block_mass(const Vec& flat) const { return apply(0, flat); }
  Vec apply_block_stiffness(const Vec& flat) const { return apply(1, flat); }
  Vec apply_block_transient(const Vec& flat) const { return apply(2, flat); }

  // sg.cpp:358-423; the ForceFn is sampled at t_0 .. t_N (the same accumulated
  // t sequence as the reference) into a nodal table
  SgHistory run(const Vec& u0_nodal, const Vec& v0_nodal, int n_steps, const ForceFn& force = nullptr) {
    if (n_steps < 0) throw std::invalid_argument("SgSolver::run: n_steps must be >= 0");
    const size_t nn = size_t(mesh_.n_nodes());
    if (u0_nodal.size() != nn || v0_nodal.size() != nn)
      throw std::invalid_argument("SgSolver::run: initial state size does not match the mesh");
    Vec table;
    sgw_force f{0, -1, 0.0, 0.0, 0.0, nullptr};
    std::vector<double> times;
    double t = 0.0;
    for (int k = 0; k <= n_steps; ++k, t += params_.dt) {
      times.push_back(t);
      if (force) {
        const Vec fk = force(t);
        if (fk.size() != nn) throw std::invalid_argument("ForceFn: nodal load size does not match the mesh");
        table.insert(table.end(), fk.begin(), fk.end());
      }
    }
    if (force) f = sgw_force{2, -1, 0.0, 0.0, 0.0, table.data()};
    const int np = (int)opt_.probe_nodes.size();
    std::vector<int> its(n_steps);
    Vec res(n_steps), pm(size_t(np) * (n_steps + 1)), ps(pm.size());
    Vec full(opt_.store_full ? size_t(n_steps + 1) * n_terms_ * n_dofs_ : 0);
    Vec pc(size_t(np) * n_terms_ * (n_steps + 1));
    sgw_history h{its.data(), res.data(), np, opt_.probe_nodes.data(), pm.data(), ps.data(),
                  full.empty() ? nullptr : full.data(), pc.empty() ? nullptr : pc.data()};
    detail::check(sgw_run(h_, u0_nodal.data(), v0_nodal.data(), n_steps, &f, &h));
    SgHistory out;
    out.times = times;
    for (int p = 0; p < np; ++p) {
      out.probe_mean.emplace_back(pm.begin() + size_t(p) * (n_steps + 1), pm.begin() + size_t(p + 1) * (n_steps + 1));
      out.probe_std.emplace_back(ps.begin() + size_t(p) * (n_steps + 1), ps.begin() + size_t(p + 1) * (n_steps + 1));
      out.probe_coeffs.emplace_back();
      for (int j = 0; j < n_terms_; ++j) {
        const size_t o = (size_t(p) * n_terms_ + j) * (n_steps + 1);
        out.probe_coeffs.back().emplace_back(pc.begin() + o, pc.begin() + o + n_steps + 1);
      }
    }
    const size_t N = size_t(n_terms_) * n_dofs_;
    for (size_t k = 0; !full.empty() && k <= (size_t)n_steps; ++k)
      out.full_state.emplace_back(full.begin() + k * N, full.begin() + (k + 1) * N);
    for (int k = 0; k < n_steps; ++k) {
      PcgReport r;
      r.iterations = its[k], r.converged = true, r.residual_history = {res[k]};
      out.reports.push_back(r);
    }
    return out;
  }

 private:
  Vec apply(int op, const Vec& x) const {
    Vec y(x.size());
    detail::check(sgw_apply_block(h_, op, x.data(), y.data()));
    return y;
  }
  StructuredMesh mesh_;
  NewmarkParams params_;
  SgOptions opt_;
  sgw_solver* h_ = nullptr;
  long long n_dofs_ = 0, n_global_ = 0, n_coarse_ = 0;
  int n_terms_ = 0;
};

// ------------------------------------------------------------- outputs ---
// The solve-sg data files (experiments.cpp:393-434, docs/outputs.md:19-30) in
// the reference's CsvWriter format (%.17g, io.cpp:15-44).  Returns file names.
inline std::string format_double(double v) {
  char b[32];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}
inline std::vector<std::string> write_sg_outputs(const std::string& dir, const SgHistory& h, int nx, int ny,
                                                 double dt, const std::vector<double>& snapshot_times = {}) {
  std::vector<std::string> names;
  auto write = [&](const std::string& name, const std::string& text) {
    FILE* f = std::fopen((dir + "/" + name).c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write " + dir + "/" + name);
    std::fwrite(text.data(), 1, text.size(), f);
    std::fclose(f);
    names.push_back(name);
  };
  auto row = [](std::initializer_list<double> a, const Vec* more = nullptr) {
    std::string r;
    for (double v : a) r += (r.empty() ? "" : ",") + format_double(v);
    if (more)
      for (double v : *more) r += "," + format_double(v);
    return r + "\n";
  };
  for (size_t p = 0; p < h.probe_mean.size(); ++p) {
    const size_t nt = p < h.probe_coeffs.size() ? h.probe_coeffs[p].size() : 0;
    std::string t = "t,mean,std";
    for (size_t j = 0; j < nt; ++j) t += ",u" + std::to_string(j);
    t += "\n";
    for (size_t s = 0; s < h.times.size(); ++s) {
      Vec c(nt);
      for (size_t j = 0; j < nt; ++j) c[j] = h.probe_coeffs[p][j][s];
      t += row({h.times[s], h.probe_mean[p][s], h.probe_std[p][s]}, &c);
    }
    write("probe_" + std::to_string(p) + ".csv", t);
  }
  if (!h.reports.empty()) {
    std::string t = "step,iterations,final_residual\n";
    for (size_t s = 0; s < h.reports.size(); ++s)
      t += row({double(s + 1), double(h.reports[s].iterations),
                h.reports[s].residual_history.empty() ? 0.0 : h.reports[s].residual_history.back()});
    write("iterations.csv", t);
  }
  if (!snapshot_times.empty() && !h.full_state.empty()) {
    const long long n = (long long)(nx - 1) * (ny - 1), nodes = (long long)(nx + 1) * (ny + 1);
    for (size_t k = 0; k < snapshot_times.size(); ++k) {
      const int step = std::min<int>((int)h.full_state.size() - 1, (int)std::llround(snapshot_times[k] / dt));
      const Vec& u = h.full_state[step];
      const int nt = int(u.size() / n);
      std::string t = "node_id,x,y,mean,std\n";
      for (long long i = 0; i < nodes; ++i) {
        const int gi = int(i % (nx + 1)), gj = int(i / (nx + 1));
        double mean = 0.0, sd = 0.0;
        if (gi > 0 && gi < nx && gj > 0 && gj < ny) {  // moments (sg.cpp:17-26), Dirichlet nodes 0
          const long long d = (long long)(gj - 1) * (nx - 1) + gi - 1;
          double var = 0.0;
          for (int j = 1; j < nt; ++j) var += u[j * n + d] * u[j * n + d];
          mean = u[d], sd = std::sqrt(var);
        }
        t += row({double(i), double(gi) / nx, double(gj) / ny, mean, sd});
      }
      write("snapshot_" + std::to_string(k) + ".csv", t);
    }
  }
  return names;
}

}  // namespace sgwave::b200
