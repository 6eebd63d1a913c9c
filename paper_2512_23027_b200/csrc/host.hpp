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
//
// Multi-GPU sharding: the ranks form an rx x ry grid and rank
// (bx, by) owns the 2D block of subdomains [ceil(bx px/rx), ceil((bx+1) px/rx))
// x [ceil(by py/ry), ...), which keeps the cut interface short.  Each rank
// numbers only the interface nodes its subdomains touch ("local interface",
// ascending global position); nodes on a rank-block boundary are held by every
// rank that touches them (<= 4, diagonal neighbours included) and their sums
// are completed by a point-to-point halo exchange (Halo).  World size 1: the
// local interface is the global one.
struct Halo {
  std::vector<int> peers;      // ranks sharing >= 1 interface node, ascending
  std::vector<int> peer_off;   // peers.size() + 1: blocks of `idx`
  std::vector<int> idx;        // per peer: shared local interface positions, ascending global position
  // per shared local node (ascending local position): the ranks touching it
  // (ascending, this rank included) as sources of its sum
  std::vector<int> node, src_ptr, src_rank, src_pos;  // src_pos: position in that peer's block (-1 = own)
};

struct Geometry {
  int nx = 0, ny = 0, px = 0, py = 0, mx = 0, my = 0;
  int n = 0;  // reduced dofs (nx-1)(ny-1), row-major over interior mesh nodes
  // n_iface: LOCAL interface nodes (all of them on one rank); n_corner: global cross points
  int n_iface = 0, n_iface_global = 0, n_corner = 0;
  std::vector<int> iface_dofs;        // local interface position -> reduced dof
  std::vector<int> iface_gpos;        // local interface position -> global interface position
  std::vector<int> iface_owner;       // local interface position -> lowest rank touching it
  std::vector<int> iface_pos_of_dof;  // reduced dof -> local interface position or -1
  std::vector<int> iface_gpos_of_dof; // reduced dof -> global interface position or -1
  std::vector<int> corner_dofs, corner_pos_of_dof;  // global cross points
  int ns = 0, ns_total = 0, world = 1, rank = 0;
  int rx = 1, ry = 1, bx0 = 0, bx1 = 0, by0 = 0, by1 = 0;  // rank grid, this rank's block of subdomains
  std::vector<int> sub_gid;        // owned subdomain (local index) -> global id (row-major), ascending
  std::vector<int> gid_to_local;   // global id -> local index or -1
  int W = 0, H = 0, nl = 0;  // padded interior grid W x H, local nodes
  struct Sub {
    int sx = 0, sy = 0, ox = 0, oy = 0, mxs = 0, mys = 0;  // origin node, real cell extent
    std::vector<int> iface_lid, iface_pos, r_local, c_local, corner_pos;  // iface_pos: local interface position
    std::vector<double> w;
    std::vector<int> lid_to_p;  // -2 interior, -1 Dirichlet, else local interface index
  };
  std::vector<Sub> sub;
  Halo halo;

  static int origin(int s, int n, int p) { return (s * n + p - 1) / p; }  // ceil(s n / p)
  int rank_of_sub(int gid) const;   // owner rank of a global subdomain
  int owner_of_dof(int d) const;    // rank holding the authoritative value of reduced dof d
  int dof(int gi, int gj) const {
    return (gi >= 1 && gi <= nx - 1 && gj >= 1 && gj <= ny - 1) ? (gj - 1) * (nx - 1) + gi - 1 : -1;
  }
};
// rank grid rx x ry for `world` ranks on px x py subdomains: the factor pair
// (rx <= px, ry <= py) with the shortest cut, (rx - 1) ny + (ry - 1) nx
bool rank_grid(int nx, int ny, int px, int py, int world, int* rx, int* ry);
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
std::vector<double> kle_spectrum(double sigma, double bx, double by, int n_vars);
std::vector<std::vector<int>> pce_indices(int n_vars, int order);
int nearest_node(int nx, int ny, double x, double y);

}  // namespace sgw
