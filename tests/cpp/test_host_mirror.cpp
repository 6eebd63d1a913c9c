// Tests of the C++ host mirror (include/sgwave_b200.hpp), in the manner of the
// reference's own suites (proj/tests/test_sg.cpp, test_dd.cpp): the GPU solver
// through the C++ interface against the CPU oracle (oracle/capi.cpp, test
// infrastructure only) on identical inputs.
//   test_host_mirror cpu : builders vs oracle, argument checking and error
//                          mapping (no GPU needed)
//   test_host_mirror gpu : operator and trajectory parity with the oracle
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <cstring>
#include <string>

#include "sgwave_b200.hpp"

extern "C" {  // oracle/capi.cpp
const char* orc_last_error();
int orc_lognormal_coeff(int, int, double, double, double, double, int, int, double*, int, int*);
int orc_triple_products(int, int, int, int, int*, int*, int*, int*, int*, int*, double*);
int orc_solver_create(int, int, int, int, int, const double*, int, int, const int*, const int*, const int*,
                      const double*, double, double, double, double, double, double, double, int, int, int, void**);
void orc_solver_destroy(void*);
void orc_solver_sizes(void*, long long*);
int orc_apply_block(void*, int, const double*, double*);
int orc_schur_apply(void*, int, const double*, double*);
int orc_run(void*, const double*, const double*, int, int, double, double, double, int*, double*, double*, int,
            const int*, double*, double*);
}

namespace b = sgwave::b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                           \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(cond)) {                                                            \
      ++g_fail;                                                               \
      std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);           \
    }                                                                         \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static double rel(const b::Vec& a, const b::Vec& c) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) num += (a[i] - c[i]) * (a[i] - c[i]), den += c[i] * c[i];
  return std::sqrt(num / std::max(den, 1e-300));
}

struct Case {
  int nx = 16, px = 2, L = 2, pin = 2, pout = 2;
  double sigma = 0.3, corr = 0.5, dt = 2e-3;
};

static void cpu_tests() {
  const Case c;
  // input builders agree with the oracle (kle.cpp, lognormal.cpp, pce.cpp) to 1e-15 of the field
  const b::CoefficientField f = b::lognormal_coeff(c.nx, c.nx, c.sigma, c.corr, c.corr, c.L, c.pin);
  int n_in = 0;
  const int nn = (c.nx + 1) * (c.nx + 1);
  std::vector<double> of(size_t(f.terms.size()) * nn);
  CHECK(orc_lognormal_coeff(c.nx, c.nx, c.sigma, c.corr, c.corr, 0.0, c.L, c.pin, of.data(), (int)of.size(), &n_in) == 0);
  CHECK(n_in == (int)f.terms.size());
  double dmax = 0.0, fmax = 0.0;
  for (int i = 0; i < n_in; ++i)
    for (int d = 0; d < nn; ++d)
      dmax = std::max(dmax, std::fabs(f.terms[i][d] - of[size_t(i) * nn + d])),
      fmax = std::max(fmax, std::fabs(of[size_t(i) * nn + d]));
  CHECK(dmax <= 1e-15 * fmax);
  const b::TripleTensor t = b::triple_products(c.L, c.pin, c.pout);
  int ni, no, ne;
  CHECK(orc_triple_products(c.L, c.pin, c.pout, 0, &ni, &no, &ne, nullptr, nullptr, nullptr, nullptr) == 0);
  size_t cnt = 0;
  for (const auto& v : t.by_input) cnt += v.size();
  CHECK(ni == t.n_input && no == t.n_output && (size_t)ne == cnt);
  // argument checking: std::invalid_argument as the reference (sg.cpp:143-145, partition.cpp:50-53)
  b::NewmarkParams p;
  p.dt = c.dt;
  CHECK(throws<std::invalid_argument>([&] { b::SgSolver s({c.nx, c.nx}, {c.nx + 1, 2}, f, t, 1.0, 0.5, 0.01, p, {}); }));
  b::TripleTensor bad = t;
  bad.n_input += 1;
  CHECK(throws<std::invalid_argument>([&] { b::SgSolver s({c.nx, c.nx}, {2, 2}, f, bad, 1.0, 0.5, 0.01, p, {}); }));
  b::NewmarkParams p0;  // dt = 0
  CHECK(throws<std::invalid_argument>([&] { b::SgSolver s({c.nx, c.nx}, {2, 2}, f, t, 1.0, 0.5, 0.01, p0, {}); }));
  // output writers on a synthetic history: CsvWriter format (%.17g), step numbering from 1
  b::SgHistory h;
  h.times = {0.0, 0.1, 0.2};
  h.probe_mean = {{1.0, 0.5, 1.0 / 3.0}};
  h.probe_std = {{0.0, 0.25, 2.0}};
  h.probe_coeffs = {{{1.0, 0.5, 1.0 / 3.0}, {0.0, 0.25, -2.0}}};
  h.reports = {b::PcgReport{3, true, {1.0, 1e-11}}, b::PcgReport{4, true, {1.0, 2.5e-11}}};
  CHECK(std::system("mkdir -p build/outputs_cpu") == 0);
  const auto names = b::write_sg_outputs("build/outputs_cpu", h, 4, 4, 0.1);
  CHECK(names.size() == 2);
  std::ifstream pf("build/outputs_cpu/probe_0.csv"), itf("build/outputs_cpu/iterations.csv");
  std::string l0, l1, l2, l3, i0, i1;
  std::getline(pf, l0), std::getline(pf, l1), std::getline(pf, l2), std::getline(pf, l3);
  std::getline(itf, i0), std::getline(itf, i1);
  CHECK(l0 == "t,mean,std,u0,u1");
  CHECK(l1 == "0,1,0,1,0");
  CHECK(l3 == "0.20000000000000001,0.33333333333333331,2,0.33333333333333331,-2");
  CHECK(i0 == "step,iterations,final_residual" && i1 == "1,3,9.9999999999999994e-12");
}

static void gpu_tests() {
  const Case c;
  const b::CoefficientField f = b::lognormal_coeff(c.nx, c.nx, c.sigma, c.corr, c.corr, c.L, c.pin);
  const b::TripleTensor t = b::triple_products(c.L, c.pin, c.pout);
  b::NewmarkParams p;
  p.dt = c.dt;
  b::SgOptions o;
  o.tol = 1e-10;
  o.store_full = true;
  const b::StructuredMesh mesh{c.nx, c.nx};
  const int probe = b::nearest_node(mesh, 0.5, 0.5);
  o.probe_nodes = {probe};
  b::SgSolver s(mesh, {c.px, c.px}, f, t, 1.0, 0.5445, 0.0174, p, o);
  // the oracle on the same inputs
  std::vector<double> flat;
  for (const auto& v : f.terms) flat.insert(flat.end(), v.begin(), v.end());
  std::vector<int> ei, ej, ek;
  std::vector<double> ev;
  for (int i = 0; i < t.n_input; ++i)
    for (const auto& e : t.by_input[i]) ei.push_back(i), ej.push_back(e.j), ek.push_back(e.k), ev.push_back(e.value);
  void* oh = nullptr;
  CHECK(orc_solver_create(c.nx, c.nx, c.px, c.px, t.n_input, flat.data(), t.n_output, (int)ev.size(), ei.data(),
                          ej.data(), ek.data(), ev.data(), 1.0, 0.5445, 0.0174, 0.5, 0.25, c.dt, 1e-10, 500, 2,
                          /*precond nn2*/ 0, &oh) == 0);
  long long sz[6];
  orc_solver_sizes(oh, sz);
  CHECK(sz[1] == s.n_terms() && sz[0] == s.n_dofs() && sz[4] == s.schur().n_global());
  // block operators (test_sg.cpp:51-73, <= 1e-12)
  b::Vec x(size_t(s.n_terms()) * s.n_dofs());
  for (size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.37 * double(i) + 0.1);
  for (int op = 0; op < 3; ++op) {
    b::Vec yo(x.size());
    orc_apply_block(oh, op, x.data(), yo.data());
    const b::Vec yg = op == 0 ? s.apply_block_mass(x) : op == 1 ? s.apply_block_stiffness(x) : s.apply_block_transient(x);
    CHECK(rel(yg, yo) <= 1e-12);
  }
  // interface system (test_dd.cpp, <= 1e-10), PCG on it (pcg.cpp:7-50)
  b::Vec xi(s.schur().n_global());
  for (size_t i = 0; i < xi.size(); ++i) xi[i] = std::cos(0.11 * double(i));
  for (int w = 0; w < 2; ++w) {
    b::Vec yo(xi.size());
    orc_schur_apply(oh, w, xi.data(), yo.data());
    CHECK(rel(w == 0 ? s.schur().matvec(xi) : s.schur().apply_nn2(xi), yo) <= 1e-10);
  }
  b::Vec rhs(xi.size());
  orc_schur_apply(oh, 0, xi.data(), rhs.data());
  auto [sol, rep] = s.schur().pcg(rhs, 500);
  CHECK(rep.converged && rep.iterations > 0 && rel(sol, xi) <= 1e-8);
  // trajectory with a Ricker ForceFn (sg.cpp:358-423): iterations +-1, state 1e-8
  const int steps = 8, nn = mesh.n_nodes();
  auto ricker = [&](double tt) {
    b::Vec fv(nn, 0.0);
    const double a = M_PI * M_PI * 100.0 * (tt - 0.1) * (tt - 0.1);
    fv[probe] = (1.0 - 2.0 * a) * std::exp(-a);
    return fv;
  };
  const b::Vec z(nn, 0.0);
  const b::SgHistory h = s.run(z, z, steps, ricker);
  std::vector<int> its(steps);
  std::vector<double> res(steps), full(size_t(steps + 1) * x.size()), pm(steps + 1), ps(steps + 1);
  CHECK(orc_run(oh, z.data(), z.data(), steps, probe, 10.0, 0.1, 1.0, its.data(), res.data(), full.data(), 1, &probe,
                pm.data(), ps.data()) == 0);
  bool iters_ok = (int)h.reports.size() == steps;
  for (int k = 0; k < steps && iters_ok; ++k) iters_ok = std::abs(h.reports[k].iterations - its[k]) <= 1;
  CHECK(iters_ok);
  b::Vec gflat, oflat(full);
  for (const auto& st : h.full_state) gflat.insert(gflat.end(), st.begin(), st.end());
  CHECK(gflat.size() == oflat.size() && rel(gflat, oflat) <= 1e-8);
  CHECK(h.probe_mean.size() == 1 && rel(h.probe_mean[0], pm) <= 1e-8);
  CHECK(h.mean_iterations() > 0.0);
  // probe chaos coefficients = the state at the probe dof (sg.cpp:391-405)
  const int pd = (probe / (c.nx + 1) - 1) * (c.nx - 1) + probe % (c.nx + 1) - 1;
  bool coeff_ok = h.probe_coeffs.size() == 1 && (int)h.probe_coeffs[0].size() == s.n_terms();
  for (int j = 0; j < s.n_terms() && coeff_ok; ++j)
    for (int k = 0; k <= steps && coeff_ok; ++k)
      coeff_ok = h.probe_coeffs[0][j][k] == h.full_state[k][size_t(j) * s.n_dofs() + pd];
  CHECK(coeff_ok);
  // solve-sg outputs (experiments.cpp:393-434)
  const std::string dir = "build/outputs_gpu";
  CHECK(std::system(("mkdir -p " + dir).c_str()) == 0);
  const auto names = b::write_sg_outputs(dir, h, c.nx, c.nx, c.dt, {0.004, 0.1});
  CHECK(names.size() == 4);  // probe_0, iterations, snapshot_0, snapshot_1
  orc_solver_destroy(oh);
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  if (mode == "cpu") {
    cpu_tests();
    // without a GPU, constructing a valid solver reports a runtime error (no CPU fallback)
  } else if (mode == "nogpu") {
    const b::CoefficientField f = b::lognormal_coeff(8, 8, 0.2, 1.0, 1.0, 1, 1);
    const b::TripleTensor t = b::triple_products(1, 1, 1);
    b::NewmarkParams p;
    p.dt = 0.05;
    CHECK(throws<std::runtime_error>([&] { b::SgSolver s({8, 8}, {2, 2}, f, t, 1.0, 0.5, 0.01, p, {}); }));
  } else {
    gpu_tests();
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
