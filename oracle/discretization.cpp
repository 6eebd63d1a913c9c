// TEST INFRASTRUCTURE ONLY — see oracle.hpp.  Mesh, partition, Dirichlet
// reduction, CSR assembly, KLE, PCE and lognormal inputs of the reference.
#include <algorithm>
#include <cmath>
#include <limits>
#include <set>
#include <stdexcept>
#include <tuple>

#include "oracle.hpp"

namespace oracle {

// src/mesh.cpp:15-58
Mesh build_unit_square_mesh(int nx, int ny) {
  if (nx < 2 || ny < 2) throw std::invalid_argument("build_unit_square_mesh: nx, ny >= 2");
  const int npx = nx + 1, npy = ny + 1;
  Mesh m;
  m.nx = nx;
  m.ny = ny;
  m.x.resize(static_cast<size_t>(npx) * npy);
  m.y.resize(m.x.size());
  for (int j = 0; j < npy; ++j)
    for (int i = 0; i < npx; ++i) {
      m.x[j * npx + i] = static_cast<double>(i) / nx;
      m.y[j * npx + i] = static_cast<double>(j) / ny;
    }
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int a = j * npx + i, b = a + 1, c = (j + 1) * npx + i + 1, d = (j + 1) * npx + i;
      m.elements.push_back({a, b, c});
      m.elements.push_back({a, c, d});
    }
  std::set<Index> bnd;
  for (int i = 0; i < npx; ++i) {
    bnd.insert(i);
    bnd.insert((npy - 1) * npx + i);
  }
  for (int j = 0; j < npy; ++j) {
    bnd.insert(j * npx);
    bnd.insert(j * npx + npx - 1);
  }
  m.dirichlet_nodes.assign(bnd.begin(), bnd.end());
  const double dx = 1.0 / nx, dy = 1.0 / ny;
  m.h = std::sqrt(dx * dx + dy * dy);
  return m;
}

// src/mesh.cpp:83-96 (ties -> lower index)
Index nearest_node(const Mesh& mesh, double x, double y) {
  Index best = 0;
  double best_d = std::numeric_limits<double>::max();
  for (Index i = 0; i < mesh.n_nodes(); ++i) {
    const double dx = mesh.x[i] - x, dy = mesh.y[i] - y;
    const double d = dx * dx + dy * dy;
    if (d < best_d) {
      best_d = d;
      best = i;
    }
  }
  return best;
}

int Partition::multiplicity_of(Index node) const {  // src/partition.cpp:40-44
  auto it = std::lower_bound(global_interface.begin(), global_interface.end(), node);
  if (it == global_interface.end() || *it != node) return 1;
  return multiplicity[static_cast<size_t>(it - global_interface.begin())];
}

// src/partition.cpp:48-133
Partition partition_structured(const Mesh& mesh, int px, int py) {
  if (px < 1 || py < 1) throw std::invalid_argument("partition_structured: px, py >= 1");
  if (px > mesh.nx || py > mesh.ny) throw std::invalid_argument("more subdomains than cells");
  Partition p;
  p.n_sub = px * py;
  p.subdomain_elements.resize(p.n_sub);
  for (Index e = 0; e < mesh.n_elements(); ++e) {
    double cx = 0.0, cy = 0.0;
    for (int k = 0; k < 3; ++k) {
      cx += mesh.x[mesh.elements[e][k]];
      cy += mesh.y[mesh.elements[e][k]];
    }
    cx /= 3;
    cy /= 3;
    const int ci = std::min(mesh.nx - 1, static_cast<int>(cx * mesh.nx));
    const int cj = std::min(mesh.ny - 1, static_cast<int>(cy * mesh.ny));
    const int s = (cj * py / mesh.ny) * px + ci * px / mesh.nx;
    p.subdomain_elements[s].push_back(e);
  }
  std::vector<std::vector<int>> node_subs(mesh.n_nodes());
  p.subdomain_nodes.resize(p.n_sub);
  for (int s = 0; s < p.n_sub; ++s) {
    std::set<Index> nodes;
    for (Index e : p.subdomain_elements[s])
      for (int k = 0; k < 3; ++k) nodes.insert(mesh.elements[e][k]);
    p.subdomain_nodes[s].assign(nodes.begin(), nodes.end());
    for (Index n : p.subdomain_nodes[s]) node_subs[n].push_back(s);
  }
  p.interior_nodes.resize(p.n_sub);
  p.interface_nodes.resize(p.n_sub);
  for (int s = 0; s < p.n_sub; ++s)
    for (Index n : p.subdomain_nodes[s])
      (node_subs[n].size() == 1 ? p.interior_nodes[s] : p.interface_nodes[s]).push_back(n);
  for (Index n = 0; n < mesh.n_nodes(); ++n)
    if (node_subs[n].size() >= 2) {
      p.global_interface.push_back(n);
      p.multiplicity.push_back(static_cast<int>(node_subs[n].size()));
    }
  const double eps = 1e-12;  // src/partition.cpp:25-31
  for (size_t k = 0; k < p.global_interface.size(); ++k) {
    const Index n = p.global_interface[k];
    const double x = mesh.x[n], y = mesh.y[n];
    const bool on_bnd = x < eps || x > 1.0 - eps || y < eps || y > 1.0 - eps;
    if (p.multiplicity[k] > 2 || on_bnd)  // corner rule src/partition.cpp:117
      p.corner_nodes.push_back(n);
    else
      p.remaining_nodes.push_back(n);
  }
  return p;
}

// src/assembly.cpp:148-158
DirichletReduction make_dirichlet_reduction(const Mesh& mesh) {
  DirichletReduction r;
  r.node_to_dof.assign(mesh.n_nodes(), -1);
  for (Index n = 0; n < mesh.n_nodes(); ++n)
    if (!std::binary_search(mesh.dirichlet_nodes.begin(), mesh.dirichlet_nodes.end(), n)) {
      r.node_to_dof[n] = r.n_dofs();
      r.dof_to_node.push_back(n);
    }
  return r;
}

Vec DirichletReduction::reduce_vector(const Vec& nodal) const {  // src/assembly.cpp:136-140
  Vec out(n_dofs());
  for (Index d = 0; d < n_dofs(); ++d) out[d] = nodal[dof_to_node[d]];
  return out;
}

// ---------------------------------------------------------------- CSR ------
Csr Csr::from_triplets(Index rows, Index cols, std::vector<Triplet> trips) {
  // stable sort keeps insertion order among duplicates; they are then summed
  // first-to-last exactly as Eigen's collapseDuplicates does.
  std::stable_sort(trips.begin(), trips.end(), [](const Triplet& a, const Triplet& b) {
    return a.r != b.r ? a.r < b.r : a.c < b.c;
  });
  Csr m;
  m.rows = rows;
  m.cols = cols;
  m.ptr.assign(rows + 1, 0);
  for (size_t t = 0; t < trips.size();) {
    size_t u = t + 1;
    double v = trips[t].v;
    while (u < trips.size() && trips[u].r == trips[t].r && trips[u].c == trips[t].c) v += trips[u++].v;
    m.col.push_back(trips[t].c);
    m.val.push_back(v);
    m.ptr[trips[t].r + 1]++;
    t = u;
  }
  for (Index r = 0; r < rows; ++r) m.ptr[r + 1] += m.ptr[r];
  return m;
}

void Csr::apply(const double* x, double* y, double alpha, bool accumulate) const {
  for (Index r = 0; r < rows; ++r) {
    double s = 0.0;
    for (Index p = ptr[r]; p < ptr[r + 1]; ++p) s += val[p] * x[col[p]];
    y[r] = accumulate ? y[r] + alpha * s : alpha * s;
  }
}

void Csr::apply_t(const double* x, double* y) const {
  for (Index r = 0; r < rows; ++r)
    for (Index p = ptr[r]; p < ptr[r + 1]; ++p) y[col[p]] += val[p] * x[r];
}

double Csr::at(Index r, Index c) const {
  for (Index p = ptr[r]; p < ptr[r + 1]; ++p)
    if (col[p] == c) return val[p];
  return 0.0;
}

namespace {
void element_geometry(const Mesh& mesh, Index e, double& area, double b[3], double c[3]) {
  const auto& el = mesh.elements[e];
  const double x0 = mesh.x[el[0]], y0 = mesh.y[el[0]];
  const double x1 = mesh.x[el[1]], y1 = mesh.y[el[1]];
  const double x2 = mesh.x[el[2]], y2 = mesh.y[el[2]];
  const double det = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0);
  area = 0.5 * det;
  b[0] = y1 - y2;
  b[1] = y2 - y0;
  b[2] = y0 - y1;
  c[0] = x2 - x1;
  c[1] = x0 - x2;
  c[2] = x1 - x0;
}
}  // namespace

// src/assembly.cpp:31-74 followed by DirichletReduction::reduce (:121-134)
Csr assemble_stiffness_reduced(const Mesh& mesh, const Vec& coeff, const DirichletReduction& red) {
  std::vector<Triplet> trips;
  trips.reserve(static_cast<size_t>(mesh.n_elements()) * 9);
  for (Index e = 0; e < mesh.n_elements(); ++e) {
    double area, b[3], c[3];
    element_geometry(mesh, e, area, b, c);
    const auto& el = mesh.elements[e];
    const double cavg = (coeff[el[0]] + coeff[el[1]] + coeff[el[2]]) / 3.0;
    for (int a = 0; a < 3; ++a)
      for (int bb = 0; bb < 3; ++bb) {
        const Index r = red.node_to_dof[el[a]], cc = red.node_to_dof[el[bb]];
        if (r < 0 || cc < 0) continue;
        trips.push_back({r, cc, cavg * (b[a] * b[bb] + c[a] * c[bb]) / (4.0 * area)});
      }
  }
  return Csr::from_triplets(red.n_dofs(), red.n_dofs(), std::move(trips));
}

// src/assembly.cpp:76-103
Csr assemble_mass_reduced(const Mesh& mesh, double density, const DirichletReduction& red) {
  std::vector<Triplet> trips;
  for (Index e = 0; e < mesh.n_elements(); ++e) {
    double area, b[3], c[3];
    element_geometry(mesh, e, area, b, c);
    const auto& el = mesh.elements[e];
    const double m = density * area / 12.0;
    for (int a = 0; a < 3; ++a)
      for (int bb = 0; bb < 3; ++bb) {
        const Index r = red.node_to_dof[el[a]], cc = red.node_to_dof[el[bb]];
        if (r < 0 || cc < 0) continue;
        trips.push_back({r, cc, a == bb ? 2 * m : m});
      }
  }
  return Csr::from_triplets(red.n_dofs(), red.n_dofs(), std::move(trips));
}

// ---------------------------------------------------------------- PCE ------
// src/pce.cpp:19-37
std::vector<std::vector<int>> multi_indices(int n_vars, int max_order) {
  if (n_vars < 1 || max_order < 0) throw std::invalid_argument("multi_indices: bad arguments");
  std::vector<std::vector<int>> out;
  std::vector<int> cur(n_vars, 0);
  std::function<void(int, int)> emit = [&](int pos, int remaining) {
    if (pos == n_vars - 1) {
      cur[pos] = remaining;
      out.push_back(cur);
      return;
    }
    for (int a = remaining; a >= 0; --a) {
      cur[pos] = a;
      emit(pos + 1, remaining - a);
    }
  };
  for (int d = 0; d <= max_order; ++d) emit(0, d);
  return out;
}

double hermite(int n, double x) {  // src/pce.cpp:39-49
  double prev = 1.0;
  if (n == 0) return prev;
  double cur = x;
  for (int k = 1; k < n; ++k) {
    const double next = x * cur - k * prev;
    prev = cur;
    cur = next;
  }
  return cur;
}

namespace {
double factorial(int n) {
  double out = 1.0;
  for (int i = 2; i <= n; ++i) out *= i;
  return out;
}
double hermite_triple(int a, int b, int c) {  // src/pce.cpp:60-67
  const int total = a + b + c;
  if (total % 2 != 0) return 0.0;
  const int s = total / 2;
  if (s < a || s < b || s < c) return 0.0;
  return factorial(a) * factorial(b) * factorial(c) /
         (factorial(s - a) * factorial(s - b) * factorial(s - c));
}
}  // namespace

// src/pce.cpp:96-122 with the order_in <= order_out guard (:97-99) LIFTED.
TripleTensor triple_products(int n_vars, int order_in, int order_out) {
  const auto in = multi_indices(n_vars, order_in);
  const auto out = multi_indices(n_vars, order_out);
  TripleTensor t;
  t.n_input = static_cast<int>(in.size());
  t.n_output = static_cast<int>(out.size());
  t.by_input.resize(in.size());
  for (size_t i = 0; i < in.size(); ++i)
    for (size_t j = 0; j < out.size(); ++j)
      for (size_t k = j; k < out.size(); ++k) {
        double value = 1.0;
        for (int v = 0; v < n_vars && value != 0.0; ++v) {
          const int a = in[i][v], b = out[j][v], c = out[k][v];
          value *= hermite_triple(a, b, c) / std::sqrt(factorial(a) * factorial(b) * factorial(c));
        }
        if (value != 0.0) t.by_input[i].push_back({static_cast<int>(j), static_cast<int>(k), value});
      }
  return t;
}

// src/pce.cpp:124-185: quadrature cross-check (Golub-Welsch by Jacobi rotations)
TripleTensor triple_products_quadrature(int n_vars, int order_in, int order_out) {
  const auto in = multi_indices(n_vars, order_in);
  const auto out = multi_indices(n_vars, order_out);
  const int np = (order_in + 2 * order_out) / 2 + 2;
  // symmetric tridiagonal Jacobi matrix, eigen-decomposed with cyclic Jacobi
  std::vector<double> A(np * np, 0.0), V(np * np, 0.0);
  for (int i = 0; i < np; ++i) V[i * np + i] = 1.0;
  for (int i = 1; i < np; ++i) A[i * np + i - 1] = A[(i - 1) * np + i] = std::sqrt(double(i));
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < np; ++p)
      for (int q = p + 1; q < np; ++q) off += A[p * np + q] * A[p * np + q];
    if (off < 1e-30) break;
    for (int p = 0; p < np; ++p)
      for (int q = p + 1; q < np; ++q) {
        const double apq = A[p * np + q];
        if (std::abs(apq) < 1e-300) continue;
        const double theta = (A[q * np + q] - A[p * np + p]) / (2 * apq);
        const double tt = (theta >= 0 ? 1 : -1) / (std::abs(theta) + std::sqrt(theta * theta + 1));
        const double cs = 1 / std::sqrt(tt * tt + 1), sn = tt * cs;
        for (int k = 0; k < np; ++k) {
          const double akp = A[k * np + p], akq = A[k * np + q];
          A[k * np + p] = cs * akp - sn * akq;
          A[k * np + q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < np; ++k) {
          const double apk = A[p * np + k], aqk = A[q * np + k];
          A[p * np + k] = cs * apk - sn * aqk;
          A[q * np + k] = sn * apk + cs * aqk;
        }
        for (int k = 0; k < np; ++k) {
          const double vkp = V[k * np + p], vkq = V[k * np + q];
          V[k * np + p] = cs * vkp - sn * vkq;
          V[k * np + q] = sn * vkp + cs * vkq;
        }
      }
  }
  std::vector<double> x(np), w(np);
  for (int i = 0; i < np; ++i) {
    x[i] = A[i * np + i];
    w[i] = V[0 * np + i] * V[0 * np + i];
  }
  const int max_order = std::max(order_in, order_out);
  std::vector<double> table((max_order + 1) * np);
  for (int a = 0; a <= max_order; ++a)
    for (int q = 0; q < np; ++q) table[a * np + q] = hermite(a, x[q]) / std::sqrt(factorial(a));
  TripleTensor t;
  t.n_input = static_cast<int>(in.size());
  t.n_output = static_cast<int>(out.size());
  t.by_input.resize(in.size());
  std::vector<int> q(n_vars, 0);
  for (size_t i = 0; i < in.size(); ++i)
    for (size_t j = 0; j < out.size(); ++j)
      for (size_t k = j; k < out.size(); ++k) {
        double acc = 0.0;
        std::fill(q.begin(), q.end(), 0);
        while (true) {
          double term = 1.0;
          for (int v = 0; v < n_vars; ++v)
            term *= w[q[v]] * table[in[i][v] * np + q[v]] * table[out[j][v] * np + q[v]] *
                    table[out[k][v] * np + q[v]];
          acc += term;
          int v = 0;
          while (v < n_vars && ++q[v] == np) q[v++] = 0;
          if (v == n_vars) break;
        }
        if (std::abs(acc) > 1e-12) t.by_input[i].push_back({int(j), int(k), acc});
      }
  return t;
}

// ---------------------------------------------------------------- KLE ------
namespace {
constexpr double kHalfWidth = 0.5;
double bisect(double lo, double hi, const std::function<double(double)>& f) {  // src/kle.cpp:16-38
  double flo = f(lo);
  const double fhi = f(hi);
  if (flo == 0.0) return lo;
  if (fhi == 0.0) return hi;
  if ((flo > 0.0) == (fhi > 0.0)) throw std::runtime_error("kle_eigens_1d: bracket failure");
  for (int it = 0; it < 200 && hi - lo > 1e-14 * hi; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double fmid = f(mid);
    if (fmid == 0.0) return mid;
    if ((fmid > 0.0) == (flo > 0.0)) {
      lo = mid;
      flo = fmid;
    } else {
      hi = mid;
    }
  }
  return 0.5 * (lo + hi);
}
}  // namespace

// src/kle.cpp:40-68
std::vector<Kle1dMode> kle_eigens_1d(double b, int n_modes) {
  if (b <= 0.0) throw std::invalid_argument("kle_eigens_1d: correlation length must be positive");
  const double c = 1.0 / b, T = kHalfWidth;
  const auto f_even = [&](double w) { return std::tan(w * T) - c / w; };
  const auto f_odd = [&](double w) { return std::tan(w * T) + w / c; };
  const auto pole = [&](int k) { return (0.5 + k) * M_PI / T; };
  std::vector<Kle1dMode> modes;
  const double nudge = 1e-9;
  modes.push_back({bisect(nudge * pole(0), pole(0) * (1.0 - nudge), f_even), 0.0, true});
  for (int m = 1; static_cast<int>(modes.size()) < n_modes; ++m) {
    const double lo = pole(m - 1), hi = pole(m), width = hi - lo;
    modes.push_back({bisect(lo + nudge * width, hi - nudge * width, f_odd), 0.0, false});
    if (static_cast<int>(modes.size()) < n_modes)
      modes.push_back({bisect(lo + nudge * width, hi - nudge * width, f_even), 0.0, true});
  }
  modes.resize(n_modes);
  for (Kle1dMode& m : modes) m.lambda = 2.0 * c / (m.omega * m.omega + c * c);
  return modes;
}

double kle_eigenfunction_1d(const Kle1dMode& mode, double x) {  // src/kle.cpp:70-78
  const double T = kHalfWidth, xc = x - 0.5, w = mode.omega;
  if (mode.even) return std::cos(w * xc) / std::sqrt(T + std::sin(2.0 * w * T) / (2.0 * w));
  return std::sin(w * xc) / std::sqrt(T - std::sin(2.0 * w * T) / (2.0 * w));
}

// src/kle.cpp:80-133 (2D tensor modes, sorted by lambda desc with (i,j) tie-break)
KleExpansion kle_exponential(double sigma, double bx, double by, int n_modes, const Mesh& mesh,
                             double mean) {
  if (sigma < 0.0) throw std::invalid_argument("kle_exponential: sigma must be nonnegative");
  if (n_modes < 1) throw std::invalid_argument("kle_exponential: need at least one mode");
  KleExpansion kle;
  kle.sigma = sigma;
  kle.bx = bx;
  kle.by = by;
  kle.mean = mean;
  const auto ex = kle_eigens_1d(bx, n_modes);
  const auto ey = (by == bx) ? ex : kle_eigens_1d(by, n_modes);
  struct Pair {
    int i, j;
    double lambda;
  };
  std::vector<Pair> pairs;
  for (int i = 0; i < n_modes; ++i)
    for (int j = 0; j < n_modes; ++j) pairs.push_back({i, j, ex[i].lambda * ey[j].lambda});
  std::sort(pairs.begin(), pairs.end(), [](const Pair& a, const Pair& b) {
    if (a.lambda != b.lambda) return a.lambda > b.lambda;
    return std::tie(a.i, a.j) < std::tie(b.i, b.j);
  });
  pairs.resize(n_modes);
  for (const Pair& p : pairs) {
    KleMode mode;
    mode.lambda = sigma * sigma * p.lambda;
    mode.phi.resize(mesh.n_nodes());
    for (Index n = 0; n < mesh.n_nodes(); ++n)
      mode.phi[n] = kle_eigenfunction_1d(ex[p.i], mesh.x[n]) * kle_eigenfunction_1d(ey[p.j], mesh.y[n]);
    kle.modes.push_back(std::move(mode));
  }
  return kle;
}

// src/lognormal.cpp:8-40
CoefficientField lognormal_pce(const KleExpansion& kle, int n_vars, int p_in) {
  if (n_vars != static_cast<int>(kle.modes.size()))
    throw std::invalid_argument("lognormal_pce: basis variables != KLE modes");
  const Index nn = static_cast<Index>(kle.modes[0].phi.size());
  std::vector<Vec> g(n_vars, Vec(nn));
  for (int v = 0; v < n_vars; ++v) {
    const double s = std::sqrt(kle.modes[v].lambda);
    for (Index x = 0; x < nn; ++x) g[v][x] = s * kle.modes[v].phi[x];
  }
  Vec c0(nn);
  for (Index x = 0; x < nn; ++x) {
    double sum_sq = 0.0;
    for (int v = 0; v < n_vars; ++v) sum_sq += g[v][x] * g[v][x];
    c0[x] = std::exp(kle.mean + 0.5 * sum_sq);
  }
  CoefficientField f;
  for (const auto& alpha : multi_indices(n_vars, p_in)) {
    Vec term = c0;
    for (int v = 0; v < n_vars; ++v) {
      double norm = 1.0;
      for (int a = 2; a <= alpha[v]; ++a) norm *= a;
      if (alpha[v] > 0) {
        const double sn = std::sqrt(norm);
        for (Index x = 0; x < nn; ++x) term[x] *= std::pow(g[v][x], double(alpha[v])) / sn;
      }
    }
    f.terms.push_back(std::move(term));
  }
  return f;
}

}  // namespace oracle
