// Host-side model of the structured SG problem: inputs, interface layout and
// the per-subdomain stencil data that the GPU setup consumes.
#pragma once

#include <array>
#include <vector>

namespace sgw {

// TripleTensor (include/sgwave/pce.hpp:24-40): entries with j <= k.
struct TensorHost {
  int n_in = 0, n_out = 0;
  std::vector<int> i, j, k;
  std::vector<double> v;
};

struct Problem {
  int nx = 0, ny = 0, px = 0, py = 0, mx = 0, my = 0;
  int n_in = 0, nt = 0;
  std::vector<double> coeff;  // n_in x n_nodes
  TensorHost tensor;
  double density = 1, alpha0 = 0, alpha1 = 0, gamma = 0.5, zeta = 0.25, dt = 0, tol = 1e-8;
  int max_iter = 500, device = 0, rank = 0, world = 1;
  int precond = 0;  // PrecondKind (dd.hpp:98): 0 nn2 (the SG path, sg.cpp:330), 1 nn1, 2 lumped
  int implicit_schur = 0;  // reduced-memory mode: S_s applied through the interior solve, not stored
  double mass_scale = 0, stiff_scale = 0;  // src/sg.cpp:147-148
  int n_nodes() const { return (nx + 1) * (ny + 1); }
};

// Interface layout of the structured partition (src/partition.cpp:48-133,
// src/dd.cpp:10-96).  Cell ci belongs to block column ci*px/nx (floor), so
// block column sx spans nodes [ox(sx), ox(sx+1)], ox(sx) = ceil(sx*nx/px);
// ragged splits (px not dividing nx) give blocks of two widths.  Every
// subdomain lives in a padded frame of mx x my cells (mx = ceil(nx/px)):
// local node lid = jl*(mx+1) + il, real nodes il <= mxs, jl <= mys, padding
// nodes beyond are inert (class -1, like Dirichlet nodes).  Interior nodes:
// 0<il<mxs, 0<jl<mys (block row jl-1, position il-1).  Interface nodes: the
// block boundary minus Dirichlet nodes, ordered by reduced dof id.
struct Geometry {
  int nx = 0, ny = 0, px = 0, py = 0, mx = 0, my = 0;
  int n = 0;  // reduced dofs (nx-1)(ny-1), row-major over interior mesh nodes
  int n_iface = 0, n_corner = 0;
  std::vector<int> iface_dofs, corner_dofs;
  std::vector<int> iface_pos_of_dof, corner_pos_of_dof;
  // multi-GPU sharding: this rank owns subdomains [s0, s0 + ns) of ns_total
  // (contiguous row-major ranges, owner_of_sub); sub[] holds the owned ones.
  int ns = 0, s0 = 0, ns_total = 0, world = 1;
  int W = 0, H = 0, nl = 0;  // padded interior grid W x H, local nodes
  struct Sub {
    int sx = 0, sy = 0, ox = 0, oy = 0, mxs = 0, mys = 0;  // origin node, real cell extent
    std::vector<int> iface_lid, iface_pos, r_local, c_local, corner_pos;
    std::vector<double> w;
    std::vector<int> lid_to_p;  // -2 interior, -1 Dirichlet, else local interface index
  };
  std::vector<Sub> sub;

  static int origin(int s, int n, int p) { return (s * n + p - 1) / p; }  // ceil(s n / p)
  static int first_sub(int r, int ns_total, int world) { return int((long long)ns_total * r / world); }
  int owner_of_sub(int s) const {
    int r = 0;
    while (r + 1 < world && first_sub(r + 1, ns_total, world) <= s) ++r;
    return r;
  }
  // rank holding the authoritative value of reduced dof d (interface: rank 0)
  int owner_of_dof(int d) const;
  int dof(int gi, int gj) const {
    return (gi >= 1 && gi <= nx - 1 && gj >= 1 && gj <= ny - 1) ? (gj - 1) * (nx - 1) + gi - 1 : -1;
  }
};
Geometry build_geometry(int nx, int ny, int px, int py, int rank = 0, int world = 1);

// P1 stencils.  K: 3 components per node (diag, E, N); the NE coupling of the
// right-diagonal P1 stiffness is exactly zero (asserted during assembly).
// M: 4 components (diag, E, N, NE).
struct Stencils {
  std::vector<double> Kg;  // [(i*3 + c) * n + d]         global reduced (assembly.cpp:31-74)
  std::vector<double> Mg;  // [c * n + d]                  global reduced (assembly.cpp:76-103)
  std::vector<double> Kl;  // [((s*n_in + i)*3 + c) * nl + lid]  local (sg.cpp:38-101)
  std::vector<double> Ml;  // [(s*4 + c) * nl + lid]
};
Stencils build_stencils(const Problem& p, const Geometry& g, bool need_local);

// Input builders (host).  src/kle.cpp, src/lognormal.cpp, src/pce.cpp, src/mesh.cpp
std::vector<std::vector<double>> lognormal_coeff(int nx, int ny, double sigma, double bx, double by,
                                                 double g0, int n_vars, int p_in);
TensorHost triple_products(int n_vars, int p_in, int p_out);
int nearest_node(int nx, int ny, double x, double y);

}  // namespace sgw
