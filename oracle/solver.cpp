// TEST INFRASTRUCTURE ONLY — see oracle.hpp.  Interface layout, local Schur
// system with the NN2 preconditioner, PCG and the SG Newmark solver.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <stdexcept>
#include <string>

#include "oracle.hpp"

namespace oracle {

namespace {
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
double norm2(const Vec& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}
double dotv(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
// y = A x for column-major dense A
void gemv(const Dense& A, const double* x, double* y) {
  std::fill(y, y + A.rows, 0.0);
  for (Index c = 0; c < A.cols; ++c) {
    const double xc = x[c];
    const double* col = &A.a[static_cast<size_t>(c) * A.rows];
#pragma omp simd
    for (Index r = 0; r < A.rows; ++r) y[r] += col[r] * xc;
  }
}
// y = A^T x
void gemv_t(const Dense& A, const double* x, double* y) {
  for (Index c = 0; c < A.cols; ++c) {
    const double* col = &A.a[static_cast<size_t>(c) * A.rows];
    double s = 0.0;
#pragma omp simd reduction(+ : s)
    for (Index r = 0; r < A.rows; ++r) s += col[r] * x[r];
    y[c] = s;
  }
}
}  // namespace

// src/dd.cpp:10-64
InterfaceLayout build_interface_layout(const Partition& part, const DirichletReduction& red) {
  InterfaceLayout L;
  std::vector<Index> iface_pos_of_dof(red.n_dofs(), -1), corner_pos_of_dof(red.n_dofs(), -1);
  for (Index node : part.global_interface)
    if (red.node_to_dof[node] >= 0) L.iface_dofs.push_back(red.node_to_dof[node]);
  std::sort(L.iface_dofs.begin(), L.iface_dofs.end());
  for (size_t q = 0; q < L.iface_dofs.size(); ++q) iface_pos_of_dof[L.iface_dofs[q]] = Index(q);
  for (Index node : part.corner_nodes)
    if (red.node_to_dof[node] >= 0) L.corner_dofs.push_back(red.node_to_dof[node]);
  std::sort(L.corner_dofs.begin(), L.corner_dofs.end());
  for (size_t q = 0; q < L.corner_dofs.size(); ++q) corner_pos_of_dof[L.corner_dofs[q]] = Index(q);
  L.sub.resize(part.n_sub);
  for (int s = 0; s < part.n_sub; ++s) {
    SubdomainDofs& sd = L.sub[s];
    for (Index node : part.interior_nodes[s])
      if (red.node_to_dof[node] >= 0) sd.interior.push_back(red.node_to_dof[node]);
    for (Index node : part.interface_nodes[s])
      if (red.node_to_dof[node] >= 0) sd.iface.push_back(red.node_to_dof[node]);
    std::sort(sd.interior.begin(), sd.interior.end());
    std::sort(sd.iface.begin(), sd.iface.end());
    sd.weights.resize(sd.iface.size());
    for (size_t k = 0; k < sd.iface.size(); ++k) {
      const Index dof = sd.iface[k];
      sd.iface_pos.push_back(iface_pos_of_dof[dof]);
      sd.weights[k] = 1.0 / part.multiplicity_of(red.dof_to_node[dof]);
      if (corner_pos_of_dof[dof] >= 0) {
        sd.c_local.push_back(Index(k));
        sd.corner_pos.push_back(corner_pos_of_dof[dof]);
      } else {
        sd.r_local.push_back(Index(k));
      }
    }
    sd.loc_dofs = sd.interior;
    sd.loc_dofs.insert(sd.loc_dofs.end(), sd.iface.begin(), sd.iface.end());
  }
  return L;
}

// src/dd.cpp:78-96
LocalSchur make_flat_maps(const SubdomainDofs& sd, int n_blocks, Index n_iface, Index n_corner) {
  LocalSchur ls;
  const Index ng = sd.n_iface(), nc = Index(sd.c_local.size());
  ls.weights.resize(size_t(n_blocks) * ng);
  for (int j = 0; j < n_blocks; ++j) {
    for (Index p = 0; p < ng; ++p) {
      ls.gmap.push_back(j * n_iface + sd.iface_pos[p]);
      ls.weights[j * ng + p] = sd.weights[p];
    }
    for (Index r : sd.r_local) ls.r_idx.push_back(j * ng + r);
    for (Index c = 0; c < nc; ++c) {
      ls.c_idx.push_back(j * ng + sd.c_local[c]);
      ls.corner_gmap.push_back(j * n_corner + sd.corner_pos[c]);
    }
  }
  return ls;
}

// src/dd.cpp:98-140
void SchurSystem::finalize(bool build_nn1) {
  const int ns = int(locals.size());
  std::vector<Dense> coarse(ns);
  parallel_for(ns, n_threads, [&](int s) {
    LocalSchur& ls = locals[s];
    const Index nr = Index(ls.r_idx.size()), nc = Index(ls.c_idx.size());
    Dense srr(nr, nr), scc(nc, nc);
    ls.S_rc = Dense(nr, nc);
    for (Index b = 0; b < nr; ++b)
      for (Index a = 0; a < nr; ++a) srr(a, b) = ls.S(ls.r_idx[a], ls.r_idx[b]);
    for (Index b = 0; b < nc; ++b)
      for (Index a = 0; a < nr; ++a) ls.S_rc(a, b) = ls.S(ls.r_idx[a], ls.c_idx[b]);
    for (Index b = 0; b < nc; ++b)
      for (Index a = 0; a < nc; ++a) scc(a, b) = ls.S(ls.c_idx[a], ls.c_idx[b]);
    ls.Srr_llt = llt_regularized(srr);
    if (build_nn1) ls.S_llt = llt_regularized(ls.S);
    if (nc > 0) {
      coarse[s] = scc;
      if (nr > 0) {
        Vec col(nr), prod(nc);
        for (Index b = 0; b < nc; ++b) {  // S_cc - S_rc^T S_rr^{-1} S_rc
          for (Index a = 0; a < nr; ++a) col[a] = ls.S_rc(a, b);
          ls.Srr_llt.solve_in_place(col.data());
          gemv_t(ls.S_rc, col.data(), prod.data());
          for (Index a = 0; a < nc; ++a) coarse[s](a, b) -= prod[a];
        }
      }
    }
  });
  if (n_corner > 0) {
    fcc_ = Dense(n_corner, n_corner);
    for (int s = 0; s < ns; ++s) {
      const LocalSchur& ls = locals[s];
      const Index nc = Index(ls.c_idx.size());
      for (Index a = 0; a < nc; ++a)
        for (Index b = 0; b < nc; ++b) fcc_(ls.corner_gmap[a], ls.corner_gmap[b]) += coarse[s](a, b);
    }
    fcc_llt_ = llt_regularized(fcc_);
    has_coarse_ = true;
  }
}

// src/dd.cpp:142-157
Vec SchurSystem::matvec(const Vec& x) const {
  const int ns = int(locals.size());
  std::vector<Vec> contrib(ns);
  parallel_for(ns, n_threads, [&](int s) {
    const LocalSchur& ls = locals[s];
    Vec xl(ls.n_flat());
    for (Index k = 0; k < ls.n_flat(); ++k) xl[k] = x[ls.gmap[k]];
    contrib[s].resize(ls.n_flat());
    gemv(ls.S, xl.data(), contrib[s].data());
  });
  Vec y(n_global, 0.0);
  for (int s = 0; s < ns; ++s)
    for (Index k = 0; k < locals[s].n_flat(); ++k) y[locals[s].gmap[k]] += contrib[s][k];
  return y;
}

// src/dd.cpp:159-176 and :178-195: z = sum_s R_s^T D_s A_s D_s R_s r with
// A_s = K~_GG,s (lumped, the solver's gg_action) or S_s^-1 (NN1)
template <typename F>
static Vec one_level(const SchurSystem& sys, const Vec& r, F&& local) {
  const int ns = int(sys.locals.size());
  std::vector<Vec> contrib(ns);
  parallel_for(ns, sys.n_threads, [&](int s) {
    const LocalSchur& ls = sys.locals[s];
    Vec rl(ls.n_flat());
    for (Index k = 0; k < ls.n_flat(); ++k) rl[k] = r[ls.gmap[k]] * ls.weights[k];
    Vec zl = local(ls, rl);
    for (Index k = 0; k < ls.n_flat(); ++k) zl[k] *= ls.weights[k];
    contrib[s] = std::move(zl);
  });
  Vec z(sys.n_global, 0.0);
  for (int s = 0; s < ns; ++s)
    for (Index k = 0; k < sys.locals[s].n_flat(); ++k) z[sys.locals[s].gmap[k]] += contrib[s][k];
  return z;
}

Vec SchurSystem::apply_lumped(const Vec& r) const {
  return one_level(*this, r, [](const LocalSchur& ls, const Vec& rl) {
    if (ls.Kgg.rows != ls.n_flat()) throw std::invalid_argument("lumped preconditioner: K~_GG not assembled");
    Vec zl(rl.size());
    gemv(ls.Kgg, rl.data(), zl.data());
    return zl;
  });
}

Vec SchurSystem::apply_nn1(const Vec& r) const {
  return one_level(*this, r, [](const LocalSchur& ls, const Vec& rl) {
    if (ls.S_llt.n != ls.n_flat()) throw std::invalid_argument("nn1 preconditioner: S_s not factored");
    Vec zl = rl;
    ls.S_llt.solve_in_place(zl.data());
    return zl;
  });
}

Vec SchurSystem::apply(int kind, const Vec& r) const {
  return kind == 1 ? apply_nn1(r) : kind == 2 ? apply_lumped(r) : apply_nn2(r);
}

// src/dd.cpp:199-253
Vec SchurSystem::apply_nn2(const Vec& r) const {
  const int ns = int(locals.size());
  std::vector<Vec> t(ns), dc(ns);
  parallel_for(ns, n_threads, [&](int s) {
    const LocalSchur& ls = locals[s];
    const Index nr = Index(ls.r_idx.size()), nc = Index(ls.c_idx.size());
    Vec rl(ls.n_flat());
    for (Index k = 0; k < ls.n_flat(); ++k) rl[k] = r[ls.gmap[k]] * ls.weights[k];
    t[s].resize(nr);
    for (Index a = 0; a < nr; ++a) t[s][a] = rl[ls.r_idx[a]];
    if (nr > 0) ls.Srr_llt.solve_in_place(t[s].data());
    if (nc > 0) {
      dc[s].resize(nc);
      for (Index a = 0; a < nc; ++a) dc[s][a] = rl[ls.c_idx[a]];
      if (nr > 0) {
        Vec prod(nc);
        gemv_t(ls.S_rc, t[s].data(), prod.data());
        for (Index a = 0; a < nc; ++a) dc[s][a] -= prod[a];
      }
    }
  });
  Vec uc;
  if (has_coarse_) {
    Vec d(n_corner, 0.0);
    for (int s = 0; s < ns; ++s)
      for (size_t a = 0; a < locals[s].corner_gmap.size(); ++a) d[locals[s].corner_gmap[a]] += dc[s][a];
    fcc_llt_.solve_in_place(d.data());
    uc = std::move(d);
  }
  std::vector<Vec> contrib(ns);
  parallel_for(ns, n_threads, [&](int s) {
    const LocalSchur& ls = locals[s];
    const Index nr = Index(ls.r_idx.size()), nc = Index(ls.c_idx.size());
    Vec zl(ls.n_flat(), 0.0), ur = t[s];
    if (has_coarse_ && nc > 0) {
      Vec ucl(nc);
      for (Index a = 0; a < nc; ++a) ucl[a] = uc[ls.corner_gmap[a]];
      if (nr > 0) {
        Vec tmp(nr);
        gemv(ls.S_rc, ucl.data(), tmp.data());
        ls.Srr_llt.solve_in_place(tmp.data());
        for (Index a = 0; a < nr; ++a) ur[a] -= tmp[a];
      }
      for (Index a = 0; a < nc; ++a) zl[ls.c_idx[a]] = ucl[a];
    }
    for (Index a = 0; a < nr; ++a) zl[ls.r_idx[a]] = ur[a];
    for (Index k = 0; k < ls.n_flat(); ++k) zl[k] *= ls.weights[k];
    contrib[s] = std::move(zl);
  });
  Vec z(n_global, 0.0);
  for (int s = 0; s < ns; ++s)
    for (Index k = 0; k < locals[s].n_flat(); ++k) z[locals[s].gmap[k]] += contrib[s][k];
  return z;
}

// src/pcg.cpp:7-50
Vec pcg(const LinearOp& op, const LinearOp& precond, const Vec& rhs, double tol, int max_iter,
        PcgReport* report) {
  PcgReport rep;
  Vec x(rhs.size(), 0.0);
  const double bnorm = norm2(rhs);
  if (bnorm == 0.0) {
    rep.converged = true;
    rep.residual_history.push_back(0.0);
    if (report) *report = rep;
    return x;
  }
  Vec r = rhs, z = precond(r), p = z;
  double rz = dotv(r, z);
  rep.residual_history.push_back(1.0);
  for (int it = 0; it < max_iter; ++it) {
    const Vec ap = op(p);
    const double alpha = rz / dotv(p, ap);
    for (size_t i = 0; i < x.size(); ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * ap[i];
    }
    ++rep.iterations;
    double rel = norm2(r) / bnorm;
    if (rel <= tol) {
      const Vec ax = op(x);
      Vec rt(rhs.size());
      for (size_t i = 0; i < rt.size(); ++i) rt[i] = rhs[i] - ax[i];
      rel = norm2(rt) / bnorm;
      rep.residual_history.push_back(rel);
      if (rel <= tol) {
        rep.converged = true;
        if (report) *report = rep;
        return x;
      }
      r = rt;
    } else {
      rep.residual_history.push_back(rel);
    }
    z = precond(r);
    const double rz_next = dotv(r, z);
    for (size_t i = 0; i < p.size(); ++i) p[i] = z[i] + (rz_next / rz) * p[i];
    rz = rz_next;
  }
  if (report) *report = rep;
  return x;
}

double SgHistory::mean_iterations() const {
  if (reports.empty()) return 0.0;
  double s = 0.0;
  for (const auto& r : reports) s += r.iterations;
  return s / reports.size();
}

// ------------------------------------------------------------ SgSolver -----
namespace {
// Local element assembly on local slots (src/sg.cpp:38-101).
void assemble_local_terms(const Mesh& mesh, const Partition& part, const DirichletReduction& red,
                          const SubdomainDofs& sd, const CoefficientField& coeff, double density,
                          int s, Csr& mass, std::vector<Csr>& k_terms) {
  std::vector<Index> slot(red.n_dofs(), -1);
  for (size_t k = 0; k < sd.loc_dofs.size(); ++k) slot[sd.loc_dofs[k]] = Index(k);
  const Index nl = Index(sd.loc_dofs.size());
  const int n_in = coeff.n_terms();
  std::vector<Triplet> tm;
  std::vector<std::vector<Triplet>> tk(n_in);
  for (Index e : part.subdomain_elements[s]) {
    const auto& el = mesh.elements[e];
    const double x0 = mesh.x[el[0]], y0 = mesh.y[el[0]], x1 = mesh.x[el[1]], y1 = mesh.y[el[1]];
    const double x2 = mesh.x[el[2]], y2 = mesh.y[el[2]];
    const double det = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0);
    const double area = 0.5 * det;
    const double b[3] = {y1 - y2, y2 - y0, y0 - y1}, c[3] = {x2 - x1, x0 - x2, x1 - x0};
    double geom[3][3];
    for (int a = 0; a < 3; ++a)
      for (int bb = 0; bb < 3; ++bb) geom[a][bb] = (b[a] * b[bb] + c[a] * c[bb]) / (4.0 * area);
    const double m = density * area / 12.0;
    for (int a = 0; a < 3; ++a) {
      const Index da = red.node_to_dof[el[a]];
      if (da < 0) continue;
      for (int bb = 0; bb < 3; ++bb) {
        const Index db = red.node_to_dof[el[bb]];
        if (db < 0) continue;
        tm.push_back({slot[da], slot[db], a == bb ? 2 * m : m});
        for (int i = 0; i < n_in; ++i) {
          double cavg = 0.0;
          for (int v = 0; v < 3; ++v) cavg += coeff.terms[i][el[v]];
          cavg /= 3;
          tk[i].push_back({slot[da], slot[db], cavg * geom[a][bb]});
        }
      }
    }
  }
  mass = Csr::from_triplets(nl, nl, std::move(tm));
  k_terms.resize(n_in);
  for (int i = 0; i < n_in; ++i) k_terms[i] = Csr::from_triplets(nl, nl, std::move(tk[i]));
}

// Extract block [r0, r0+nr) x [c0, c0+nc) as triplets (src/sg.cpp:117-130).
void block_triplets(const Csr& m, Index r0, Index nr, Index c0, Index nc, Index row_off,
                    Index col_off, double scale, std::vector<Triplet>& out) {
  for (Index r = r0; r < r0 + nr; ++r)
    for (Index p = m.ptr[r]; p < m.ptr[r + 1]; ++p) {
      const Index c = m.col[p];
      if (c >= c0 && c < c0 + nc) out.push_back({row_off + r - r0, col_off + c - c0, scale * m.val[p]});
    }
}

// Node-band half-width of a square CSR operator.
Index node_bandwidth(const Csr& m) {
  Index bw = 0;
  for (Index r = 0; r < m.rows; ++r)
    for (Index p = m.ptr[r]; p < m.ptr[r + 1]; ++p) bw = std::max(bw, std::abs(r - m.col[p]));
  return bw;
}

// Band factor of a term-major flattened SG operator over `nn` nodes: the band
// index of flat (term j, node k) is k*nt + j.  `entries` are the CSR blocks
// that make up the operator in reference triplet order.
bool factor_flattened(const std::vector<Triplet>& trips, Index nn, int nt, Index node_bw,
                      BandLlt& llt) {
  const Index n = nn * nt, bw = node_bw * nt + (nt - 1);
  Csr a = Csr::from_triplets(n, n, trips);  // rows in term-major flat index
  // build node-major rows: band row i = (k, j) <- flat row j*nn + k
  return llt.compute(n, bw, [&](Index i, double* row) {
    const Index k = i / nt, j = i % nt, fr = j * nn + k;
    for (Index p = a.ptr[fr]; p < a.ptr[fr + 1]; ++p) {
      const Index fc = a.col[p];
      const Index bc = (fc % nn) * nt + fc / nn;
      if (bc <= i && bc >= i - bw) row[bc - i + bw] = a.val[p];
    }
  });
}

void to_band(const double* flat, double* band, Index nn, int nt) {
  for (int j = 0; j < nt; ++j)
    for (Index k = 0; k < nn; ++k) band[k * nt + j] = flat[j * nn + k];
}
void from_band(const double* band, double* flat, Index nn, int nt) {
  for (int j = 0; j < nt; ++j)
    for (Index k = 0; k < nn; ++k) flat[j * nn + k] = band[k * nt + j];
}
}  // namespace

// src/sg.cpp:128-176
SgSolver::SgSolver(const Mesh& mesh, const Partition& part, const CoefficientField& coeff,
                   const TripleTensor& tensor, double density, double alpha0, double alpha1,
                   NewmarkParams params, SgOptions options)
    : mesh_(mesh),
      part_(part),
      red_(make_dirichlet_reduction(mesh)),
      layout_(build_interface_layout(part, red_)),
      coeff_(coeff),
      tensor_(tensor),
      n_terms_(tensor.n_output),
      density_(density),
      alpha0_(alpha0),
      alpha1_(alpha1),
      params_(params),
      opt_(std::move(options)) {
  const double t0 = now_s();
  if (coeff.n_terms() != tensor.n_input)
    throw std::invalid_argument("SgSolver: coefficient terms do not match tensor input size");
  direct_ = part.n_sub == 1 || layout_.n_iface() == 0;
  mass_scale_ = params_.mass_factor() + params_.damping_factor() * alpha0_;
  stiff_scale_ = 1.0 + params_.damping_factor() * alpha1_;
  mass_red_ = assemble_mass_reduced(mesh, density, red_);
  const Index n = red_.n_dofs();
  const Index nbw = node_bandwidth(mass_red_);
  {
    std::vector<Triplet> t;
    block_triplets(mass_red_, 0, n, 0, n, 0, 0, 1.0, t);
    if (!factor_flattened(t, n, 1, nbw, mass_llt_)) throw std::runtime_error("mass factorization failed");
  }
  for (int i = 0; i < coeff.n_terms(); ++i) k_red_.push_back(assemble_stiffness_reduced(mesh, coeff.terms[i], red_));
  if (direct_) {
    std::vector<Triplet> t;
    for (int j = 0; j < n_terms_; ++j) block_triplets(mass_red_, 0, n, 0, n, j * n, j * n, mass_scale_, t);
    for (int i = 0; i < tensor_.n_input; ++i)
      tensor_.for_each(i, [&](int j, int k, double g) {
        block_triplets(k_red_[i], 0, n, 0, n, k * n, j * n, stiff_scale_ * g, t);
      });
    if (!factor_flattened(t, n, n_terms_, nbw, direct_llt_))
      throw std::runtime_error("stochastic transient stiffness factorization failed");
  } else {
    assemble_subdomains();
  }
  t_setup = now_s() - t0;
}

// src/sg.cpp:178-250
void SgSolver::assemble_subdomains() {
  const int ns = part_.n_sub, nt = n_terms_;
  locals_.resize(ns);
  schur_.n_global = nt * layout_.n_iface();
  schur_.n_corner = nt * layout_.n_corner();
  schur_.n_threads = opt_.threads;
  schur_.locals.resize(ns);
  const Ctx cx{mesh_, part_, red_, layout_, coeff_, tensor_, density_, mass_scale_, stiff_scale_, nt, opt_.precond};
  parallel_for(ns, opt_.threads, [&](int s) { build_local(cx, s, 1, locals_[s], schur_.locals[s]); });
  schur_.finalize(opt_.precond == 1);
}

// The body of assemble_subdomains' per-subdomain loop (src/sg.cpp:186-246):
// local terms, flattened A_II / A_IG, the interior factor and the dense local
// Schur S = A_GG - A_IG^T A_II^-1 A_IG.  panel_threads > 1 splits the
// right-hand-side panels of the elimination over threads (independent columns).
void SgSolver::build_local(const Ctx& cx, int s, int panel_threads, Local& loc, LocalSchur& ls) {
  const int nt = cx.nt;
  const SubdomainDofs& sd = cx.layout.sub[s];
  assemble_local_terms(cx.mesh, cx.part, cx.red, sd, cx.coeff, cx.density, s, loc.mass, loc.k_terms);
  const Index ni = sd.n_interior(), ng = sd.n_iface();
  // flattened interior block and interior x iface coupling (src/sg.cpp:203-217)
  std::vector<Triplet> t_ii, t_ig;
  for (int j = 0; j < nt; ++j) {
    block_triplets(loc.mass, 0, ni, 0, ni, j * ni, j * ni, cx.mass_scale, t_ii);
    block_triplets(loc.mass, 0, ni, ni, ng, j * ni, j * ng, cx.mass_scale, t_ig);
  }
  for (int i = 0; i < cx.tensor.n_input; ++i)
    cx.tensor.for_each(i, [&](int j, int k, double g) {
      block_triplets(loc.k_terms[i], 0, ni, 0, ni, k * ni, j * ni, cx.stiff_scale * g, t_ii);
      block_triplets(loc.k_terms[i], 0, ni, ni, ng, k * ni, j * ng, cx.stiff_scale * g, t_ig);
    });
  loc.a_ig = Csr::from_triplets(nt * ni, nt * ng, std::move(t_ig));
  if (ni > 0) {
    // node band of the interior block
    Index nbw = 0;
    for (Index r = 0; r < ni; ++r)
      for (Index p = loc.mass.ptr[r]; p < loc.mass.ptr[r + 1]; ++p)
        if (loc.mass.col[p] < ni) nbw = std::max(nbw, std::abs(r - loc.mass.col[p]));
    for (const Csr& kt : loc.k_terms)
      for (Index r = 0; r < ni; ++r)
        for (Index p = kt.ptr[r]; p < kt.ptr[r + 1]; ++p)
          if (kt.col[p] < ni) nbw = std::max(nbw, std::abs(r - kt.col[p]));
    if (!factor_flattened(t_ii, ni, nt, nbw, loc.ii))
      throw std::runtime_error("stochastic interior factorization failed (subdomain " + std::to_string(s) + ")");
    loc.has_interior = true;
  }
  // dense flattened local Schur (src/sg.cpp:227-245)
  ls = make_flat_maps(sd, nt, cx.layout.n_iface(), cx.layout.n_corner());
  const Index a = nt * ng;
  ls.S = Dense(a, a);
  for (int j = 0; j < nt; ++j)
    for (Index r = 0; r < ng; ++r)
      for (Index p = loc.mass.ptr[ni + r]; p < loc.mass.ptr[ni + r + 1]; ++p) {
        const Index c = loc.mass.col[p];
        if (c >= ni) ls.S(j * ng + r, j * ng + c - ni) += cx.mass_scale * loc.mass.val[p];
      }
  for (int i = 0; i < cx.tensor.n_input; ++i) {
    const Csr& kt = loc.k_terms[i];
    cx.tensor.for_each(i, [&](int j, int k, double g) {
      const double sg = cx.stiff_scale * g;
      for (Index r = 0; r < ng; ++r)
        for (Index p = kt.ptr[ni + r]; p < kt.ptr[ni + r + 1]; ++p) {
          const Index c = kt.col[p];
          if (c >= ni) ls.S(k * ng + r, j * ng + c - ni) += sg * kt.val[p];
        }
    });
  }
  if (cx.precond == 2) ls.Kgg = ls.S;  // A_GG before the elimination
  if (ni > 0 && ng > 0) {
    // S -= A_IG^T A_II^{-1} A_IG, panels of RHS in band index space, columns
    // ordered by their first non-zero band row so panels skip leading zeros.
    const Index nb = nt * ni;
    std::vector<std::vector<std::pair<Index, double>>> cols(a);  // band-row entries per column
    for (Index fr = 0; fr < nb; ++fr)
      for (Index p = loc.a_ig.ptr[fr]; p < loc.a_ig.ptr[fr + 1]; ++p) {
        const Index br = (fr % ni) * nt + fr / ni;
        cols[loc.a_ig.col[p]].push_back({br, loc.a_ig.val[p]});
      }
    std::vector<Index> order(a), first(a, nb);
    for (Index c = 0; c < a; ++c) {
      order[c] = c;
      for (auto& e : cols[c]) first[c] = std::min(first[c], e.first);
    }
    std::stable_sort(order.begin(), order.end(), [&](Index x, Index y) { return first[x] < first[y]; });
    const Index P = 32;
    const int n_panels = int((a + P - 1) / P);
    // each panel updates only its own columns of S: panels are independent
    parallel_for(n_panels, panel_threads, [&](int pi) {
      const Index c0 = Index(pi) * P;
      const Index w = std::min(P, a - c0);
      std::vector<double> panel(size_t(nb) * w, 0.0);
      for (Index q = 0; q < w; ++q)
        for (auto& e : cols[order[c0 + q]]) panel[size_t(e.first) * w + q] = e.second;
      loc.ii.solve_many(panel.data(), w);
      // S(c', order[c0+q]) -= sum_r A_IG(r, c') X(r, q)
      for (Index fr = 0; fr < nb; ++fr) {
        const Index br = (fr % ni) * nt + fr / ni;
        const double* xr = &panel[size_t(br) * w];
        for (Index p = loc.a_ig.ptr[fr]; p < loc.a_ig.ptr[fr + 1]; ++p) {
          const Index cp = loc.a_ig.col[p];
          const double v = loc.a_ig.val[p];
          for (Index q = 0; q < w; ++q) ls.S(cp, order[c0 + q]) -= v * xr[q];
        }
      }
    });
  }
}

// One subdomain's local operators without the rest of the solver: S_s (as
// assemble_subdomains builds it), S_rr^{-1} V for caller vectors V, and
// Psi = S_rr^{-1} S_rc (src/dd.cpp:112-120).  Used to check the GPU's
// per-subdomain tiles at sizes where the whole oracle exceeds host memory.
LocalSchur SgSolver::local_blocks(const Mesh& mesh, const Partition& part, const CoefficientField& coeff,
                                  const TripleTensor& tensor, double density, double alpha0, double alpha1,
                                  NewmarkParams params, int s, int threads) {
  const DirichletReduction red = make_dirichlet_reduction(mesh);
  const InterfaceLayout layout = build_interface_layout(part, red);
  if (s < 0 || s >= part.n_sub) throw std::invalid_argument("subdomain out of range");
  const double ms = params.mass_factor() + params.damping_factor() * alpha0;
  const double ss = 1.0 + params.damping_factor() * alpha1;
  const Ctx cx{mesh, part, red, layout, coeff, tensor, density, ms, ss, tensor.n_output, 0};
  Local loc;
  LocalSchur ls;
  build_local(cx, s, threads, loc, ls);
  const Index nr = Index(ls.r_idx.size()), nc = Index(ls.c_idx.size());
  Dense srr(nr, nr);
  ls.S_rc = Dense(nr, nc);
  for (Index b = 0; b < nr; ++b)
    for (Index a = 0; a < nr; ++a) srr(a, b) = ls.S(ls.r_idx[a], ls.r_idx[b]);
  for (Index b = 0; b < nc; ++b)
    for (Index a = 0; a < nr; ++a) ls.S_rc(a, b) = ls.S(ls.r_idx[a], ls.c_idx[b]);
  ls.Srr_llt = llt_regularized(srr);
  return ls;
}

void SgSolver::interior_solve(int s, double* flat) const {
  const Local& loc = locals_[s];
  const Index ni = layout_.sub[s].n_interior();
  std::vector<double> band(size_t(ni) * n_terms_);
  to_band(flat, band.data(), ni, n_terms_);
  loc.ii.solve_in_place(band.data());
  from_band(band.data(), flat, ni, n_terms_);
}

// src/sg.cpp:252-293
Vec SgSolver::local_force(int s, const Vec& um, const Vec& uc, const Vec& f_next) const {
  const SubdomainDofs& sd = layout_.sub[s];
  const Local& loc = locals_[s];
  const Index n = red_.n_dofs(), nl = Index(sd.loc_dofs.size()), ni = sd.n_interior(), ng = sd.n_iface();
  const int nt = n_terms_;
  std::vector<Vec> umc(nt, Vec(nl)), ucl(nt, Vec(nl)), f(nt, Vec(nl));
  for (int j = 0; j < nt; ++j)
    for (Index k = 0; k < nl; ++k) {
      const double um_v = um[size_t(j) * n + sd.loc_dofs[k]], uc_v = uc[size_t(j) * n + sd.loc_dofs[k]];
      umc[j][k] = um_v + alpha0_ * uc_v;
      ucl[j][k] = uc_v;
    }
  for (int j = 0; j < nt; ++j) loc.mass.apply(umc[j].data(), f[j].data());
  if (alpha1_ > 0.0) {
    Vec tmp(nl);
    for (int i = 0; i < tensor_.n_input; ++i)
      tensor_.for_each(i, [&](int j, int k, double g) {
        loc.k_terms[i].apply(ucl[j].data(), tmp.data());
        const double sc = alpha1_ * g;
        for (Index r = 0; r < nl; ++r) f[k][r] += sc * tmp[r];
      });
  }
  if (!f_next.empty()) {
    for (Index k = 0; k < ni; ++k) f[0][k] += f_next[sd.interior[k]];
    for (Index k = 0; k < ng; ++k) f[0][ni + k] += sd.weights[k] * f_next[sd.iface[k]];
  }
  Vec flat(size_t(nt) * nl);
  for (int j = 0; j < nt; ++j) {
    for (Index k = 0; k < ni; ++k) flat[size_t(j) * ni + k] = f[j][k];
    for (Index k = 0; k < ng; ++k) flat[size_t(nt) * ni + size_t(j) * ng + k] = f[j][ni + k];
  }
  return flat;
}

// src/sg.cpp:295-356
Vec SgSolver::step_rhs_and_solve(const StateTriple& st, const Vec& f_next, PcgReport* report) {
  const Index n = red_.n_dofs();
  const int nt = n_terms_;
  const size_t N = size_t(nt) * n;
  const double dt = params_.dt, zeta = params_.zeta, gamma = params_.gamma;
  Vec um(N), uc(N);
  const double cm = (1.0 - 2.0 * zeta) / (2.0 * zeta), zdd = zeta * dt * dt;  // src/newmark.cpp:16-26
  for (size_t i = 0; i < N; ++i) um[i] = (st.u[i] + dt * st.v[i]) / zdd + cm * st.a[i];
  for (size_t i = 0; i < N; ++i) uc[i] = gamma * dt * um[i] - st.v[i] - (1.0 - gamma) * dt * st.a[i];
  if (direct_) {
    Vec rhs = apply_block_mass(um);
    const Vec mc = apply_block_mass(uc), kc = apply_block_stiffness(uc);
    for (size_t i = 0; i < N; ++i) rhs[i] = rhs[i] + alpha0_ * mc[i] + alpha1_ * kc[i];
    if (!f_next.empty())
      for (Index i = 0; i < n; ++i) rhs[i] += f_next[i];
    Vec band(N);
    to_band(rhs.data(), band.data(), n, nt);
    direct_llt_.solve_in_place(band.data());
    from_band(band.data(), rhs.data(), n, nt);
    return rhs;
  }
  const int ns = part_.n_sub;
  std::vector<Vec> g_contrib(ns), y_int(ns);
  parallel_for(ns, opt_.threads, [&](int s) {
    const SubdomainDofs& sd = layout_.sub[s];
    const Local& loc = locals_[s];
    const Index ni = sd.n_interior(), ng = sd.n_iface();
    const Vec f = local_force(s, um, uc, f_next);
    Vec g(f.begin() + size_t(nt) * ni, f.end());
    if (ni > 0) {
      y_int[s].assign(f.begin(), f.begin() + size_t(nt) * ni);
      interior_solve(s, y_int[s].data());
      Vec aty(size_t(nt) * ng, 0.0);  // g -= A_IG^T y (src/sg.cpp:318)
      loc.a_ig.apply_t(y_int[s].data(), aty.data());
      for (size_t k = 0; k < g.size(); ++k) g[k] -= aty[k];
    }
    g_contrib[s] = std::move(g);
  });
  Vec g_iface(schur_.n_global, 0.0);
  for (int s = 0; s < ns; ++s) {
    const LocalSchur& ls = schur_.locals[s];
    for (Index k = 0; k < ls.n_flat(); ++k) g_iface[ls.gmap[k]] += g_contrib[s][k];
  }
  const double tp = now_s();
  const LinearOp mv = [this](const Vec& x) { return schur_.matvec(x); };
  const LinearOp pc = [this](const Vec& r) { return schur_.apply(opt_.precond, r); };
  const Vec u_iface = pcg(mv, pc, g_iface, opt_.tol, opt_.max_iter, report);
  t_pcg += now_s() - tp;
  Vec u_next(N);
  const Index n_ifc = layout_.n_iface();
  for (int j = 0; j < nt; ++j)
    for (Index q = 0; q < n_ifc; ++q) u_next[size_t(j) * n + layout_.iface_dofs[q]] = u_iface[size_t(j) * n_ifc + q];
  parallel_for(ns, opt_.threads, [&](int s) {
    const SubdomainDofs& sd = layout_.sub[s];
    const Local& loc = locals_[s];
    const Index ni = sd.n_interior(), ng = sd.n_iface();
    if (ni == 0) return;
    Vec ug(size_t(nt) * ng), w(size_t(nt) * ni);
    for (int j = 0; j < nt; ++j)
      for (Index k = 0; k < ng; ++k) ug[size_t(j) * ng + k] = u_iface[size_t(j) * n_ifc + sd.iface_pos[k]];
    loc.a_ig.apply(ug.data(), w.data());
    interior_solve(s, w.data());
    for (int j = 0; j < nt; ++j)
      for (Index k = 0; k < ni; ++k)
        u_next[size_t(j) * n + sd.interior[k]] = y_int[s][size_t(j) * ni + k] - w[size_t(j) * ni + k];
  });
  return u_next;
}

// src/sg.cpp:358-423
SgHistory SgSolver::run(const Vec& u0_nodal, const Vec& v0_nodal, int n_steps, const ForceFn& force) {
  const double t0 = now_s();
  t_pcg = 0.0;
  total_iterations = 0;
  const Index n = red_.n_dofs();
  const int nt = n_terms_;
  const size_t N = size_t(nt) * n;
  StateTriple st;
  st.u.assign(N, 0.0);
  st.v.assign(N, 0.0);
  {
    const Vec u0 = red_.reduce_vector(u0_nodal), v0 = red_.reduce_vector(v0_nodal);
    std::copy(u0.begin(), u0.end(), st.u.begin());
    std::copy(v0.begin(), v0.end(), st.v.begin());
  }
  Vec f0(N, 0.0);
  if (force) {
    const Vec f = red_.reduce_vector(force(0.0));
    std::copy(f.begin(), f.end(), f0.begin());
  }
  const Vec mv = apply_block_mass(st.v), kv = apply_block_stiffness(st.v), ku = apply_block_stiffness(st.u);
  Vec resid(N);
  for (size_t i = 0; i < N; ++i) resid[i] = f0[i] - alpha0_ * mv[i] - alpha1_ * kv[i] - ku[i];
  st.a.resize(N);
  for (int j = 0; j < nt; ++j) {
    std::copy(resid.begin() + size_t(j) * n, resid.begin() + size_t(j + 1) * n, st.a.begin() + size_t(j) * n);
    mass_llt_.solve_in_place(st.a.data() + size_t(j) * n);
  }
  st.t = 0.0;
  std::vector<Index> probe_dofs;
  for (Index node : opt_.probe_nodes) {
    const Index dof = red_.node_to_dof[node];
    if (dof < 0) throw std::invalid_argument("probe node is constrained");
    probe_dofs.push_back(dof);
  }
  SgHistory h;
  h.probe_mean.assign(probe_dofs.size(), {});
  h.probe_std.assign(probe_dofs.size(), {});
  auto record = [&](const StateTriple& s) {
    h.times.push_back(s.t);
    for (size_t p = 0; p < probe_dofs.size(); ++p) {
      double var = 0.0;
      for (int j = 1; j < nt; ++j) {
        const double c = s.u[size_t(j) * n + probe_dofs[p]];
        var += c * c;
      }
      h.probe_mean[p].push_back(s.u[probe_dofs[p]]);
      h.probe_std[p].push_back(std::sqrt(var));
    }
    if (opt_.store_full) h.full_state.push_back(s.u);
  };
  record(st);
  const double dt = params_.dt, zeta = params_.zeta, gamma = params_.gamma;
  const double zdd = zeta * dt * dt, cm = (1.0 - 2.0 * zeta) / (2.0 * zeta);
  for (int step = 0; step < n_steps; ++step) {
    Vec f_next;
    if (force) f_next = red_.reduce_vector(force(st.t + dt));
    PcgReport rep;
    const Vec u_next = step_rhs_and_solve(st, f_next, direct_ ? nullptr : &rep);
    if (!direct_) {
      if (!rep.converged)
        throw std::runtime_error("stochastic interface solve did not converge at step " + std::to_string(step));
      total_iterations += rep.iterations;
      h.reports.push_back(std::move(rep));
    }
    // src/newmark.cpp:39-49
    StateTriple nx;
    nx.u = u_next;
    nx.a.resize(N);
    nx.v.resize(N);
    for (size_t i = 0; i < N; ++i) nx.a[i] = (u_next[i] - st.u[i] - dt * st.v[i]) / zdd - cm * st.a[i];
    for (size_t i = 0; i < N; ++i) nx.v[i] = st.v[i] + (1.0 - gamma) * dt * st.a[i] + gamma * dt * nx.a[i];
    nx.t = st.t + dt;
    st = std::move(nx);
    record(st);
  }
  t_steps = now_s() - t0;
  return h;
}

// src/sg.cpp:425-447
Vec SgSolver::apply_block_mass(const Vec& flat) const {
  const Index n = red_.n_dofs();
  Vec out(size_t(n_terms_) * n);
  for (int j = 0; j < n_terms_; ++j) mass_red_.apply(flat.data() + size_t(j) * n, out.data() + size_t(j) * n);
  return out;
}
Vec SgSolver::apply_block_stiffness(const Vec& flat) const {
  const Index n = red_.n_dofs();
  Vec out(size_t(n_terms_) * n, 0.0), tmp(n);
  for (int i = 0; i < tensor_.n_input; ++i)
    tensor_.for_each(i, [&](int j, int k, double g) {
      k_red_[i].apply(flat.data() + size_t(j) * n, tmp.data());
      double* o = out.data() + size_t(k) * n;
      for (Index r = 0; r < n; ++r) o[r] += g * tmp[r];
    });
  return out;
}
Vec SgSolver::apply_block_transient(const Vec& flat) const {
  const Vec m = apply_block_mass(flat), k = apply_block_stiffness(flat);
  Vec out(m.size());
  for (size_t i = 0; i < m.size(); ++i) out[i] = mass_scale_ * m[i] + stiff_scale_ * k[i];
  return out;
}

}  // namespace oracle
