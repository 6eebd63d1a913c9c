// Host-side inputs and structured layout for the GPU SG solver.
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>
#include <stdexcept>
#include <thread>
#include <tuple>

#include "common.cuh"

namespace sgw {

// ----------------------------------------------------------- geometry ------
bool rank_grid(int nx, int ny, int px, int py, int world, int* rx, int* ry) {
  long long best = -1;
  for (int a = 1; a <= world; ++a) {
    if (world % a) continue;
    const int b = world / a;
    if (a > px || b > py) continue;
    const long long cut = (long long)(a - 1) * ny + (long long)(b - 1) * nx;
    if (best < 0 || cut < best || (cut == best && a > *rx)) best = cut, *rx = a, *ry = b;
  }
  return best >= 0;
}

int Geometry::rank_of_sub(int gid) const {
  const int sx = gid % px, sy = gid / px;
  int bx = 0, by = 0;
  while (bx + 1 < rx && origin(bx + 1, px, rx) <= sx) ++bx;
  while (by + 1 < ry && origin(by + 1, py, ry) <= sy) ++by;
  return by * rx + bx;
}

// Structured restatement of partition_structured (src/partition.cpp:48-133,
// floor-division cell ownership, so ragged splits are allowed) and
// build_interface_layout / make_flat_maps (src/dd.cpp:10-96): interface =
// non-Dirichlet nodes on internal block lines, corners = cross points
// (multiplicity 4; boundary-touching corners are Dirichlet).
Geometry build_geometry(int nx, int ny, int px, int py, int rank, int world) {
  if (nx < 2 || ny < 2) throw Error(1, "build_unit_square_mesh: nx and ny must be >= 2");
  if (px < 1 || py < 1 || px > nx || py > ny) throw Error(1, "partition_structured: bad px/py");
  Geometry g;
  g.nx = nx, g.ny = ny, g.px = px, g.py = py;
  g.mx = (nx + px - 1) / px, g.my = (ny + py - 1) / py;  // widest block (partition.cpp:70-76)
  // blocks of one cell (no interior dofs, test_dd.cpp:98-107) live in a frame
  // of at least 2 x 2 cells: its interior slot is then a unit row, like the
  // padding slots of a ragged block, and S_s = K~_GG
  g.mx = std::max(g.mx, 2), g.my = std::max(g.my, 2);
  g.n = (nx - 1) * (ny - 1);
  g.ns_total = px * py;
  if (world < 1 || rank < 0 || rank >= world) throw Error(1, "bad rank / world_size");
  if (world > g.ns_total) throw Error(1, "more ranks than subdomains");
  if (!rank_grid(nx, ny, px, py, world, &g.rx, &g.ry))
    throw Error(1, "world_size " + std::to_string(world) + " does not factor into a rank grid rx x ry with rx <= px, "
                   "ry <= py");
  g.world = world, g.rank = rank;
  g.bx0 = Geometry::origin(rank % g.rx, px, g.rx), g.bx1 = Geometry::origin(rank % g.rx + 1, px, g.rx);
  g.by0 = Geometry::origin(rank / g.rx, py, g.ry), g.by1 = Geometry::origin(rank / g.rx + 1, py, g.ry);
  g.gid_to_local.assign(g.ns_total, -1);
  for (int sy = g.by0; sy < g.by1; ++sy)
    for (int sx = g.bx0; sx < g.bx1; ++sx) {
      g.gid_to_local[sy * px + sx] = int(g.sub_gid.size());
      g.sub_gid.push_back(sy * px + sx);
    }
  g.ns = int(g.sub_gid.size());
  std::vector<char> vl(nx + 1, 0), hl(ny + 1, 0);
  for (int s = 1; s < px; ++s) vl[Geometry::origin(s, nx, px)] = 1;
  for (int s = 1; s < py; ++s) hl[Geometry::origin(s, ny, py)] = 1;
  // ranks touching node (gi, gj): owners of the subdomains of its <= 4 cells
  auto ranks_at = [&](int gi, int gj, int* out) {
    int c = 0;
    for (int cj = gj - 1; cj <= gj; ++cj)
      for (int ci = gi - 1; ci <= gi; ++ci) {
        if (ci < 0 || cj < 0 || ci >= nx || cj >= ny) continue;
        const int r = g.rank_of_sub((cj * py / ny) * px + ci * px / nx);
        bool seen = false;
        for (int k = 0; k < c; ++k) seen |= out[k] == r;
        if (!seen) out[c++] = r;
      }
    for (int a = 1; a < c; ++a)  // insertion sort of <= 4 ranks
      for (int b = a; b > 0 && out[b - 1] > out[b]; --b) std::swap(out[b - 1], out[b]);
    return c;
  };
  g.iface_pos_of_dof.assign(g.n, -1);
  g.iface_gpos_of_dof.assign(g.n, -1);
  g.corner_pos_of_dof.assign(g.n, -1);
  std::vector<std::vector<int>> shared_with;  // per local interface node: ranks touching it
  for (int gj = 1; gj < ny; ++gj)
    for (int gi = 1; gi < nx; ++gi) {
      const bool vline = vl[gi], hline = hl[gj];
      if (!(vline || hline)) continue;
      const int d = g.dof(gi, gj);
      g.iface_gpos_of_dof[d] = g.n_iface_global++;
      if (vline && hline) {
        g.corner_pos_of_dof[d] = static_cast<int>(g.corner_dofs.size());
        g.corner_dofs.push_back(d);
      }
      int rk[4];
      const int c = ranks_at(gi, gj, rk);
      if (!std::binary_search(rk, rk + c, rank)) continue;
      g.iface_pos_of_dof[d] = static_cast<int>(g.iface_dofs.size());
      g.iface_dofs.push_back(d);
      g.iface_gpos.push_back(g.iface_gpos_of_dof[d]);
      g.iface_owner.push_back(rk[0]);
      shared_with.emplace_back(rk, rk + c);
    }
  g.n_iface = static_cast<int>(g.iface_dofs.size());
  g.n_corner = static_cast<int>(g.corner_dofs.size());
  // halo plan: per peer the shared nodes (ascending global position = local order)
  {
    Halo& h = g.halo;
    std::vector<std::vector<int>> by_peer(world);
    for (int q = 0; q < g.n_iface; ++q)
      for (int r : shared_with[q])
        if (r != rank) by_peer[r].push_back(q);
    std::vector<int> pos_in_peer(world, -1);
    h.peer_off.push_back(0);
    for (int r = 0; r < world; ++r) {
      if (by_peer[r].empty()) continue;
      pos_in_peer[r] = int(h.peers.size());
      h.peers.push_back(r);
      h.idx.insert(h.idx.end(), by_peer[r].begin(), by_peer[r].end());
      h.peer_off.push_back(int(h.idx.size()));
    }
    h.src_ptr.push_back(0);
    std::vector<int> cursor(h.peers.size(), 0);
    for (int q = 0; q < g.n_iface; ++q) {
      if (shared_with[q].size() < 2) continue;
      h.node.push_back(q);
      for (int r : shared_with[q]) {
        h.src_rank.push_back(r);
        if (r == rank) {
          h.src_pos.push_back(-1);
        } else {  // q is the cursor-th shared node of this peer (both lists ascend)
          const int pi = pos_in_peer[r];
          h.src_pos.push_back(cursor[pi]++);
        }
      }
      h.src_ptr.push_back(int(h.src_rank.size()));
    }
  }
  g.W = g.mx - 1;
  g.H = g.my - 1;
  g.nl = (g.mx + 1) * (g.my + 1);
  g.sub.resize(g.ns);
  for (int sl = 0; sl < g.ns; ++sl) {
    Geometry::Sub& sd = g.sub[sl];
    const int s = g.sub_gid[sl];
    sd.sx = s % px;
    sd.sy = s / px;
    sd.ox = Geometry::origin(sd.sx, nx, px), sd.oy = Geometry::origin(sd.sy, ny, py);
    sd.mxs = Geometry::origin(sd.sx + 1, nx, px) - sd.ox, sd.mys = Geometry::origin(sd.sy + 1, ny, py) - sd.oy;
    sd.lid_to_p.assign(g.nl, -1);
    // ascending reduced dof id == row-major over local nodes
    for (int jl = 0; jl <= sd.mys; ++jl)
      for (int il = 0; il <= sd.mxs; ++il) {
        const int lid = jl * (g.mx + 1) + il;
        const int d = g.dof(sd.ox + il, sd.oy + jl);
        if (d < 0) continue;
        if (il > 0 && il < sd.mxs && jl > 0 && jl < sd.mys) {
          sd.lid_to_p[lid] = -2;
          continue;
        }
        const int p = static_cast<int>(sd.iface_lid.size());
        sd.lid_to_p[lid] = p;
        sd.iface_lid.push_back(lid);
        sd.iface_pos.push_back(g.iface_pos_of_dof[d]);
        const bool corner = g.corner_pos_of_dof[d] >= 0;
        sd.w.push_back(corner ? 0.25 : 0.5);  // 1 / multiplicity
        if (corner) {
          sd.c_local.push_back(p);
          sd.corner_pos.push_back(g.corner_pos_of_dof[d]);
        } else {
          sd.r_local.push_back(p);
        }
      }
  }
  return g;
}

int Geometry::owner_of_dof(int d) const {
  if (world == 1) return 0;
  if (iface_gpos_of_dof[d] >= 0) {  // interface: the lowest rank touching it
    const int gi = d % (nx - 1) + 1, gj = d / (nx - 1) + 1;
    int lo = world;
    for (int cj = gj - 1; cj <= gj; ++cj)
      for (int ci = gi - 1; ci <= gi; ++ci)
        lo = std::min(lo, rank_of_sub((cj * py / ny) * px + ci * px / nx));
    return lo;
  }
  const int gi = d % (nx - 1) + 1, gj = d / (nx - 1) + 1;
  return rank_of_sub((gj * py / ny) * px + gi * px / nx);  // interior: the block of cell (gi, gj)
}

// ----------------------------------------------------------- stencils ------
namespace {
struct Elem {
  int n[3];
};
// element geometry exactly as the reference computes it from node coordinates
void geom_of(const int gi[3], const int gj[3], int nx, int ny, double& area, double b[3], double c[3]) {
  const double x0 = double(gi[0]) / nx, y0 = double(gj[0]) / ny;
  const double x1 = double(gi[1]) / nx, y1 = double(gj[1]) / ny;
  const double x2 = double(gi[2]) / nx, y2 = double(gj[2]) / ny;
  const double det = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0);
  area = 0.5 * det;
  b[0] = y1 - y2, b[1] = y2 - y0, b[2] = y0 - y1;
  c[0] = x2 - x1, c[1] = x0 - x2, c[2] = x1 - x0;
}
// triangles of cell (ci, cj): lower (a,b,c), upper (a,c,d)  (src/mesh.cpp:38-49)
void cell_tris(int ci, int cj, int tri, int gi[3], int gj[3]) {
  const int ai = ci, aj = cj, bi = ci + 1, bj = cj, cI = ci + 1, cJ = cj + 1, di = ci, dj = cj + 1;
  if (tri == 0) {
    gi[0] = ai, gj[0] = aj, gi[1] = bi, gj[1] = bj, gi[2] = cI, gj[2] = cJ;
  } else {
    gi[0] = ai, gj[0] = aj, gi[1] = cI, gj[1] = cJ, gi[2] = di, gj[2] = dj;
  }
}
}  // namespace

Stencils build_stencils(const Problem& p, const Geometry& g, bool need_local) {
  Stencils st;
  const int n = g.n, nin = p.n_in, nn1 = p.nx + 1;
  st.Kg.assign(size_t(nin) * 3 * n, 0.0);
  st.Mg.assign(size_t(4) * n, 0.0);
  auto slot = [](int da, int db, int e_off, int n_off, int ne_off) -> int {
    const int o = db - da;
    return o == 0 ? 0 : o == e_off ? 1 : o == n_off ? 2 : o == ne_off ? 3 : -1;
  };
  // global reduced assembly, element order (assembly.cpp:31-103 + reduce :121-134)
  for (int cj = 0; cj < p.ny; ++cj)
    for (int ci = 0; ci < p.nx; ++ci)
      for (int tri = 0; tri < 2; ++tri) {
        int gi[3], gj[3];
        cell_tris(ci, cj, tri, gi, gj);
        double area, b[3], c[3];
        geom_of(gi, gj, p.nx, p.ny, area, b, c);
        const double m = p.density * area / 12.0;
        int d[3], node[3];
        for (int a = 0; a < 3; ++a) d[a] = g.dof(gi[a], gj[a]), node[a] = gj[a] * nn1 + gi[a];
        for (int a = 0; a < 3; ++a)
          for (int bb = 0; bb < 3; ++bb) {
            if (d[a] < 0 || d[bb] < 0 || d[bb] < d[a]) continue;
            const int sl = slot(d[a], d[bb], 1, p.nx - 1, p.nx);
            if (sl < 0) throw Error(1, "unexpected coupling in structured mesh");
            st.Mg[size_t(sl) * n + d[a]] += (a == bb ? 2 * m : m);
            if (sl == 3) {
              const double gg = b[a] * b[bb] + c[a] * c[bb];
              if (gg != 0.0) throw Error(1, "non-zero diagonal stiffness coupling: mesh not supported");
              continue;
            }
            for (int i = 0; i < nin; ++i) {
              const double* cf = &p.coeff[size_t(i) * p.n_nodes()];
              const double cavg = (cf[node[0]] + cf[node[1]] + cf[node[2]]) / 3.0;
              st.Kg[(size_t(i) * 3 + sl) * n + d[a]] += cavg * (b[a] * b[bb] + c[a] * c[bb]) / (4.0 * area);
            }
          }
      }
  if (!need_local) return st;
  // local assembly on each subdomain's own elements (src/sg.cpp:38-101)
  const int nl = g.nl, mx = g.mx;
  st.Kl.assign(size_t(g.ns) * nin * 3 * nl, 0.0);
  st.Ml.assign(size_t(g.ns) * 4 * nl, 0.0);
  auto work = [&](int s) {
    const Geometry::Sub& sd = g.sub[s];
    for (int cjl = 0; cjl < sd.mys; ++cjl)
      for (int cil = 0; cil < sd.mxs; ++cil)
        for (int tri = 0; tri < 2; ++tri) {
          int gi[3], gj[3];
          cell_tris(sd.ox + cil, sd.oy + cjl, tri, gi, gj);
          double area, b[3], c[3];
          geom_of(gi, gj, p.nx, p.ny, area, b, c);
          double geom[3][3];
          for (int a = 0; a < 3; ++a)
            for (int bb = 0; bb < 3; ++bb) geom[a][bb] = (b[a] * b[bb] + c[a] * c[bb]) / (4.0 * area);
          const double m = p.density * area / 12.0;
          int lid[3], node[3];
          bool free_[3];
          for (int a = 0; a < 3; ++a) {
            lid[a] = (gj[a] - sd.oy) * (mx + 1) + (gi[a] - sd.ox);
            node[a] = gj[a] * nn1 + gi[a];
            free_[a] = g.dof(gi[a], gj[a]) >= 0;
          }
          for (int a = 0; a < 3; ++a)
            for (int bb = 0; bb < 3; ++bb) {
              if (!free_[a] || !free_[bb] || lid[bb] < lid[a]) continue;
              const int sl = slot(lid[a], lid[bb], 1, mx + 1, mx + 2);
              st.Ml[(size_t(s) * 4 + sl) * nl + lid[a]] += (a == bb ? 2 * m : m);
              if (sl == 3) {
                if (geom[a][bb] != 0.0) throw Error(1, "non-zero diagonal stiffness coupling");
                continue;
              }
              for (int i = 0; i < nin; ++i) {
                const double* cf = &p.coeff[size_t(i) * p.n_nodes()];
                double cavg = 0.0;
                for (int v = 0; v < 3; ++v) cavg += cf[node[v]];
                cavg /= 3;
                st.Kl[((size_t(s) * nin + i) * 3 + sl) * nl + lid[a]] += cavg * geom[a][bb];
              }
            }
        }
  };
  const int nth = std::max(1, std::min<int>(g.ns, int(std::thread::hardware_concurrency())));
  std::vector<std::thread> th;
  for (int t = 0; t < nth; ++t)
    th.emplace_back([&, t] {
      for (int s = t; s < g.ns; s += nth) work(s);
    });
  for (auto& t : th) t.join();
  return st;
}

// ------------------------------------------------------------- inputs ------
namespace {
double fact(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= i;
  return f;
}
std::vector<std::vector<int>> graded_indices(int L, int p) {  // src/pce.cpp:19-37
  std::vector<std::vector<int>> out;
  std::vector<int> cur(L, 0);
  std::function<void(int, int)> rec = [&](int pos, int rem) {
    if (pos == L - 1) {
      cur[pos] = rem;
      out.push_back(cur);
      return;
    }
    for (int a = rem; a >= 0; --a) {
      cur[pos] = a;
      rec(pos + 1, rem - a);
    }
  };
  for (int d = 0; d <= p; ++d) rec(0, d);
  return out;
}
// <He_a He_b He_c> / sqrt(a! b! c!)  (src/pce.cpp:60-67, :108-113)
double triple_1d(int a, int b, int c) {
  const int t = a + b + c;
  if (t & 1) return 0.0;
  const int s = t / 2;
  if (s < a || s < b || s < c) return 0.0;
  return fact(a) * fact(b) * fact(c) / (fact(s - a) * fact(s - b) * fact(s - c)) /
         std::sqrt(fact(a) * fact(b) * fact(c));
}
// Roots of the exponential-kernel characteristic equations on [-1/2, 1/2] by
// bisection (src/kle.cpp:16-68).
struct Root {
  double w, lambda;
  bool even;
};
double bisect(double lo, double hi, const std::function<double(double)>& f) {
  double flo = f(lo);
  const double fhi = f(hi);
  if (flo == 0.0) return lo;
  if (fhi == 0.0) return hi;
  if ((flo > 0.0) == (fhi > 0.0)) throw Error(1, "kle: bracket failure");
  for (int it = 0; it < 200 && hi - lo > 1e-14 * hi; ++it) {
    const double mid = 0.5 * (lo + hi), fm = f(mid);
    if (fm == 0.0) return mid;
    if ((fm > 0.0) == (flo > 0.0))
      lo = mid, flo = fm;
    else
      hi = mid;
  }
  return 0.5 * (lo + hi);
}
std::vector<Root> roots_1d(double b, int n) {
  if (b <= 0.0) throw Error(1, "kle: correlation length must be positive");
  const double c = 1.0 / b, T = 0.5, nudge = 1e-9;
  auto fe = [&](double w) { return std::tan(w * T) - c / w; };
  auto fo = [&](double w) { return std::tan(w * T) + w / c; };
  auto pole = [&](int k) { return (0.5 + k) * M_PI / T; };
  std::vector<Root> r;
  r.push_back({bisect(nudge * pole(0), pole(0) * (1.0 - nudge), fe), 0, true});
  for (int m = 1; int(r.size()) < n; ++m) {
    const double lo = pole(m - 1), hi = pole(m), w = hi - lo;
    r.push_back({bisect(lo + nudge * w, hi - nudge * w, fo), 0, false});
    if (int(r.size()) < n) r.push_back({bisect(lo + nudge * w, hi - nudge * w, fe), 0, true});
  }
  r.resize(n);
  for (Root& x : r) x.lambda = 2.0 * c / (x.w * x.w + c * c);
  return r;
}
double eigfun(const Root& r, double x) {
  const double T = 0.5, xc = x - 0.5;
  return r.even ? std::cos(r.w * xc) / std::sqrt(T + std::sin(2.0 * r.w * T) / (2.0 * r.w))
                : std::sin(r.w * xc) / std::sqrt(T - std::sin(2.0 * r.w * T) / (2.0 * r.w));
}
}  // namespace

std::vector<std::vector<double>> lognormal_coeff(int nx, int ny, double sigma, double bx, double by,
                                                 double g0, int L, int p_in) {
  if (sigma < 0.0 || L < 1) throw Error(1, "kle_exponential: bad sigma / n_modes");
  const auto ex = roots_1d(bx, L);
  const auto ey = (by == bx) ? ex : roots_1d(by, L);
  struct Pr {
    int i, j;
    double l;
  };
  std::vector<Pr> pr;
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < L; ++j) pr.push_back({i, j, ex[i].lambda * ey[j].lambda});
  std::sort(pr.begin(), pr.end(), [](const Pr& a, const Pr& b) {
    if (a.l != b.l) return a.l > b.l;
    return std::tie(a.i, a.j) < std::tie(b.i, b.j);
  });
  const int nn = (nx + 1) * (ny + 1);
  std::vector<std::vector<double>> gv(L, std::vector<double>(nn));
  for (int v = 0; v < L; ++v) {
    const double sl = std::sqrt(sigma * sigma * pr[v].l);
    for (int node = 0; node < nn; ++node) {
      const double x = double(node % (nx + 1)) / nx, y = double(node / (nx + 1)) / ny;
      gv[v][node] = sl * (eigfun(ex[pr[v].i], x) * eigfun(ey[pr[v].j], y));
    }
  }
  std::vector<double> c0(nn);
  for (int x = 0; x < nn; ++x) {
    double s2 = 0.0;
    for (int v = 0; v < L; ++v) s2 += gv[v][x] * gv[v][x];
    c0[x] = std::exp(g0 + 0.5 * s2);
  }
  std::vector<std::vector<double>> out;
  for (const auto& al : graded_indices(L, p_in)) {
    std::vector<double> t = c0;
    for (int v = 0; v < L; ++v)
      if (al[v] > 0) {
        double nrm = 1.0;
        for (int a = 2; a <= al[v]; ++a) nrm *= a;
        const double sn = std::sqrt(nrm);
        for (int x = 0; x < nn; ++x) t[x] *= std::pow(gv[v][x], double(al[v])) / sn;
      }
    out.push_back(std::move(t));
  }
  return out;
}

// the first L eigenvalues sigma^2 lambda_i lambda_j of the 2D separable
// exponential covariance, sorted like kle_exponential (src/kle.cpp:80-133):
// kle_spectrum.csv's lambda column
std::vector<double> kle_spectrum(double sigma, double bx, double by, int L) {
  if (L < 1) throw Error(1, "kle_spectrum: n_modes must be >= 1");
  const auto ex = roots_1d(bx, L);
  const auto ey = (by == bx) ? ex : roots_1d(by, L);
  std::vector<std::tuple<double, int, int>> pr;
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < L; ++j) pr.emplace_back(ex[i].lambda * ey[j].lambda, i, j);
  std::sort(pr.begin(), pr.end(), [](const auto& a, const auto& b) {
    if (std::get<0>(a) != std::get<0>(b)) return std::get<0>(a) > std::get<0>(b);
    return std::tie(std::get<1>(a), std::get<2>(a)) < std::tie(std::get<1>(b), std::get<2>(b));
  });
  std::vector<double> out(L);
  for (int v = 0; v < L; ++v) out[v] = sigma * sigma * std::get<0>(pr[v]);  // KleMode::lambda
  return out;
}

std::vector<std::vector<int>> pce_indices(int n_vars, int order) {  // PceBasis order (src/pce.cpp:19-37)
  if (n_vars < 1 || order < 0) throw Error(1, "pce_indices: bad arguments");
  return graded_indices(n_vars, order);
}

// src/pce.cpp:96-122 with the order_in <= order_out guard lifted.
TensorHost triple_products(int L, int p_in, int p_out) {
  if (L < 1 || p_in < 0 || p_out < 0) throw Error(1, "triple_products: bad arguments");
  const auto in = graded_indices(L, p_in), out = graded_indices(L, p_out);
  TensorHost t;
  t.n_in = int(in.size());
  t.n_out = int(out.size());
  for (int i = 0; i < t.n_in; ++i)
    for (int j = 0; j < t.n_out; ++j)
      for (int k = j; k < t.n_out; ++k) {
        double v = 1.0;
        for (int q = 0; q < L && v != 0.0; ++q) v *= triple_1d(in[i][q], out[j][q], out[k][q]);
        if (v != 0.0) {
          t.i.push_back(i);
          t.j.push_back(j);
          t.k.push_back(k);
          t.v.push_back(v);
        }
      }
  return t;
}

int nearest_node(int nx, int ny, double x, double y) {  // src/mesh.cpp:83-96
  int best = 0;
  double bd = std::numeric_limits<double>::max();
  for (int node = 0; node < (nx + 1) * (ny + 1); ++node) {
    const double dx = double(node % (nx + 1)) / nx - x, dy = double(node / (nx + 1)) / ny - y;
    const double d = dx * dx + dy * dy;
    if (d < bd) bd = d, best = node;
  }
  return best;
}

}  // namespace sgw
