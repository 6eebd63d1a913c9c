"""ctypes mirror of the reference solver interface over libsgw_b200.so.

Names, argument meaning and error behaviour follow the reference:
  SgSolver(mesh, partition, coeff, tensor, density, alpha0, alpha1, params, options)
      include/sgwave/sg.hpp:45-47  (mesh/partition given by their structured sizes)
  SgSolver.run(u0_nodal, v0_nodal, n_steps, force) -> SgHistory   sg.hpp:49-50
  SgSolver.apply_block_mass/stiffness/transient                    sg.hpp:58-60
  SgSolver.schur().matvec / apply_nn2 / coarse_operator            dd.hpp:85-90
  SgSolver.pcg(rhs) == pcg(matvec, apply_nn2, rhs, tol, max_iter)   pcg.hpp:20-21
Errors raise SgError subclasses matching the reference exception classes:
std::invalid_argument -> ValueError, factorization / non-convergence ->
RuntimeError (see include/sgw.h).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB = None

SGW_OK, SGW_EINVAL, SGW_EFACTOR, SGW_ENOCONV, SGW_ECUDA, SGW_ENCCL, SGW_ENOMEM = range(7)


class SgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class SgInvalidArgument(SgError, ValueError):
    pass


def lib_path():
    return os.path.join(_PKG, "lib", "libsgw_b200.so")


class _Problem(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("px", C.c_int), ("py", C.c_int),
                ("n_input", C.c_int), ("coeff", C.c_void_p), ("n_output", C.c_int), ("n_entries", C.c_int),
                ("ent_i", C.c_void_p), ("ent_j", C.c_void_p), ("ent_k", C.c_void_p), ("ent_v", C.c_void_p),
                ("density", C.c_double), ("alpha0", C.c_double), ("alpha1", C.c_double),
                ("gamma", C.c_double), ("zeta", C.c_double), ("dt", C.c_double),
                ("tol", C.c_double), ("max_iter", C.c_int), ("device", C.c_int),
                ("rank", C.c_int), ("world_size", C.c_int), ("nccl_id", C.c_void_p), ("precond", C.c_int),
                ("implicit_schur", C.c_int)]


class _Force(C.Structure):
    _fields_ = [("kind", C.c_int), ("node", C.c_int), ("f0", C.c_double), ("t0", C.c_double),
                ("amp", C.c_double), ("table", C.c_void_p)]


class _History(C.Structure):
    _fields_ = [("iterations", C.c_void_p), ("residual", C.c_void_p), ("n_probes", C.c_int),
                ("probe_nodes", C.c_void_p), ("probe_mean", C.c_void_p), ("probe_std", C.c_void_p),
                ("full_state", C.c_void_p), ("probe_coeffs", C.c_void_p)]


def load_library():
    """Load libsgw_b200.so; raises if it is missing (no CPU fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    vp, ip, dp = C.c_void_p, C.c_int, C.c_double
    L.sgw_last_error.restype = C.c_char_p
    L.sgw_create.argtypes = [C.POINTER(_Problem), C.POINTER(vp)]
    L.sgw_destroy.argtypes = [vp]
    L.sgw_sizes.argtypes = [vp, vp]
    L.sgw_set_stream.argtypes = [vp, vp]
    L.sgw_apply_block.argtypes = [vp, ip, vp, vp]
    L.sgw_schur_matvec.argtypes = [vp, vp, vp]
    L.sgw_apply_nn2.argtypes = [vp, vp, vp]
    L.sgw_apply_precond.argtypes = [vp, C.c_int, vp, vp]
    L.sgw_pcg.argtypes = [vp, vp, vp, vp, vp, vp, ip]
    L.sgw_coarse_operator.argtypes = [vp, vp]
    L.sgw_local_block.argtypes = [vp, ip, ip, vp, vp, vp]
    L.sgw_run.argtypes = [vp, vp, vp, ip, C.POINTER(_Force), C.POINTER(_History)]
    L.sgw_init_state.argtypes = [vp, vp, vp, C.POINTER(_Force)]
    L.sgw_advance.argtypes = [vp, ip, vp]
    L.sgw_get_state.argtypes = [vp, vp]
    L.sgw_stats.argtypes = [vp, vp]
    L.sgw_reset_stats.argtypes = [vp]
    L.sgw_kernel_profile.argtypes = [vp, ip, vp]
    L.sgw_bench_kernel.argtypes = [vp, ip, ip, vp]
    L.sgw_lognormal_coeff.argtypes = [ip, ip, dp, dp, dp, dp, ip, ip, vp, C.c_longlong, C.POINTER(ip)]
    L.sgw_triple_products.argtypes = [ip, ip, ip, C.POINTER(ip), C.POINTER(ip), C.POINTER(ip), vp, vp, vp, vp,
                                      C.c_longlong]
    L.sgw_nearest_node.argtypes = [ip, ip, dp, dp]
    L.sgw_kle_spectrum.argtypes = [dp, dp, dp, ip, vp]
    L.sgw_schur_from_locals.argtypes = [C.c_longlong, C.c_longlong, ip, vp, C.POINTER(vp)]
    L.sgw_schur_free.argtypes = [vp]
    L.sgw_schur_free.restype = None
    for nm in ("sgw_gschur_matvec", "sgw_gschur_apply_nn2"):
        getattr(L, nm).argtypes = [vp, vp, vp]
    L.sgw_gschur_coarse_operator.argtypes = [vp, vp]
    L.sgw_gschur_pcg.argtypes = [vp, vp, dp, ip, vp, C.POINTER(ip), C.POINTER(ip), vp, ip, C.POINTER(ip)]
    L.sgw_pcg_ops.argtypes = [C.c_longlong, _HOST_OP, vp, _HOST_OP, vp, vp, dp, ip, vp, C.POINTER(ip), C.POINTER(ip), vp, ip,
                              C.POINTER(ip)]
    L.sgw_pce_indices.argtypes = [ip, ip, vp, C.c_longlong, C.POINTER(ip)]
    L.sgw_nccl_unique_id.argtypes = [vp]
    L.sgw_shard_plan.argtypes = [ip, ip, ip, ip, ip, ip, vp, vp, vp, vp, vp, vp]
    L.sgw_local_group_new.argtypes = [ip, C.POINTER(vp)]
    L.sgw_local_group_free.argtypes = [vp]
    L.sgw_local_group_abort.argtypes = [vp]
    L.sgw_create_solo.argtypes = [C.POINTER(_Problem), ip, ip, C.POINTER(vp)]
    L.sgw_create_local_group.argtypes = [C.POINTER(_Problem), ip, ip, vp, C.POINTER(vp)]
    _LIB = L
    return L


def _check(rc):
    if rc != SGW_OK:
        msg = load_library().sgw_last_error().decode()
        if rc == SGW_EINVAL:
            raise SgInvalidArgument(rc, msg)
        raise SgError(rc, msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ inputs --
@dataclass
class TripleTensor:
    """include/sgwave/pce.hpp:24-40 — entries (i, j, k, value) with j <= k."""
    n_input: int
    n_output: int
    i: np.ndarray
    j: np.ndarray
    k: np.ndarray
    v: np.ndarray


def triple_products(n_vars, order_in, order_out) -> TripleTensor:
    """src/pce.cpp:96-122, with the order_in <= order_out guard lifted."""
    L = load_library()
    ni, no, ne = C.c_int(), C.c_int(), C.c_int()
    _check(L.sgw_triple_products(n_vars, order_in, order_out, C.byref(ni), C.byref(no), C.byref(ne),
                                 None, None, None, None, 0))
    i = np.zeros(ne.value, np.int32)
    j, k, v = np.zeros_like(i), np.zeros_like(i), np.zeros(ne.value)
    _check(L.sgw_triple_products(n_vars, order_in, order_out, C.byref(ni), C.byref(no), C.byref(ne),
                                 _p(i), _p(j), _p(k), _p(v), ne.value))
    return TripleTensor(ni.value, no.value, i, j, k, v)


def lognormal_coeff(nx, ny, sigma, bx, by, n_vars, p_in, g0=0.0) -> np.ndarray:
    """lognormal_pce(kle_exponential(sigma, bx, by, n_vars, mesh, g0), PceBasis(n_vars, p_in))
    (src/lognormal.cpp:8-40, src/kle.cpp:80-133): n_in x (nx+1)(ny+1) nodal terms."""
    L = load_library()
    n_in = C.c_int()
    _check(L.sgw_lognormal_coeff(nx, ny, sigma, bx, by, g0, n_vars, p_in, None, 0, C.byref(n_in)))
    out = np.zeros((n_in.value, (nx + 1) * (ny + 1)))
    _check(L.sgw_lognormal_coeff(nx, ny, sigma, bx, by, g0, n_vars, p_in, _p(out), out.size, C.byref(n_in)))
    return out


def kle_spectrum(sigma, bx, by, n_vars) -> np.ndarray:
    """The n_vars sorted KleMode::lambda of kle_exponential (src/kle.cpp:80-133)."""
    out = np.zeros(n_vars)
    _check(load_library().sgw_kle_spectrum(sigma, bx, by, n_vars, _p(out)))
    return out


def pce_indices(n_vars, order) -> np.ndarray:
    """PceBasis(n_vars, order) multi-indices in basis order (src/pce.cpp:19-37): n_terms x n_vars."""
    L = load_library()
    n = C.c_int()
    _check(L.sgw_pce_indices(n_vars, order, None, 0, C.byref(n)))
    out = np.zeros((n.value, n_vars), np.int32)
    _check(L.sgw_pce_indices(n_vars, order, _p(out), out.size, C.byref(n)))
    return out


def nearest_node(nx, ny, x, y) -> int:
    return load_library().sgw_nearest_node(nx, ny, x, y)


def gaussian_pulse(nx, ny, x0=0.7, y0=0.7, beta=1.0, alpha=0.01):
    """src/experiments.cpp:14-22"""
    i = np.tile(np.arange(nx + 1), ny + 1) / nx
    j = np.repeat(np.arange(ny + 1), nx + 1) / ny
    return np.array([beta * math.exp(-((a - x0) ** 2 + (b - y0) ** 2) / alpha) for a, b in zip(i, j)])


def ricker(t, f0=10.0, t0=0.1, amp=1.0):
    a = math.pi ** 2 * f0 ** 2 * (t - t0) ** 2
    return amp * (1.0 - 2.0 * a) * math.exp(-a)


@dataclass
class ForceSpec:
    """ForceFn (include/sgwave/det_loop.hpp:32): a Ricker point source or a
    nodal table with one row per time level t_0 .. t_N."""
    node: int = -1
    f0: float = 10.0
    t0: float = 0.1
    amp: float = 1.0
    table: np.ndarray | None = None

    def _c(self):
        if self.table is not None:
            self._keep = _f64(self.table)
            return _Force(2, -1, 0.0, 0.0, 0.0, _p(self._keep))
        if self.node >= 0:
            return _Force(1, self.node, self.f0, self.t0, self.amp, None)
        return _Force(0, -1, 0.0, 0.0, 0.0, None)


@dataclass
class NewmarkParams:  # include/sgwave/newmark.hpp:11-19
    dt: float = 1e-3
    gamma: float = 0.5
    zeta: float = 0.25


@dataclass
class SgOptions:  # include/sgwave/sg.hpp:15-21 (+ SolveOptions::precond, det_loop.hpp:14)
    precond: str = "nn2"  # PrecondKind: "nn2" (the SG path, sg.cpp:330), "nn1", "lumped"
    implicit_schur: bool = False  # reduced-memory mode: S_s applied through the interior solve (include/sgw.h)
    tol: float = 1e-8
    max_iter: int = 500
    store_full: bool = False
    probe_nodes: list = field(default_factory=list)
    device: int = 0


@dataclass
class SgHistory:  # include/sgwave/sg.hpp:23-31
    times: np.ndarray
    iterations: np.ndarray
    residual: np.ndarray
    probe_mean: np.ndarray
    probe_std: np.ndarray
    full_state: np.ndarray | None
    probe_coeffs: np.ndarray | None = None  # n_probes x (P+1) x (n_steps+1)

    def mean_iterations(self):
        return float(self.iterations.mean()) if len(self.iterations) else 0.0


def _g17(v) -> str:
    return "%.17g" % v  # io.cpp:15-19 format_double


def _write_csv(path, header, rows):
    with open(path, "w", newline="") as f:
        f.write(header + "\n")
        for r in rows:
            f.write(",".join(_g17(v) for v in r) + "\n")


def moments(flat_state, n_dofs):
    """sg.cpp:17-26: mean = u_0, std = sqrt(sum_{j>=1} u_j^2) per dof."""
    u = np.asarray(flat_state, np.float64)
    nt = u.size // n_dofs
    var = np.zeros(n_dofs)
    for j in range(1, nt):
        var += u[j * n_dofs:(j + 1) * n_dofs] ** 2
    return u[:n_dofs].copy(), np.sqrt(var)


def kle_spectrum_csv(lambdas) -> str:
    """src/kle.cpp:161-167 (ostream precision 17)"""
    return "n,lambda\n" + "".join(f"{n + 1},{_g17(v)}\n" for n, v in enumerate(lambdas))


def pce_indices_csv(indices) -> str:
    """PceBasis::indices_csv (src/pce.cpp:84-94)"""
    return "term,total_order,exponents\n" + "".join(
        f"{k},{int(sum(a))},{';'.join(str(int(v)) for v in a)}\n" for k, a in enumerate(indices))


def svg_lines(title, xlabel, ylabel, series, logx=False, logy=False) -> str:
    """write_svg_lines (src/io.cpp:58-123): series = [(label, xs, ys)]; numbers in
    the ostream default format (%g)."""
    width, height, ml, mr, mt, mb = 720, 480, 70, 160, 40, 50
    def ax(v, lg):
        return math.log10(v) if lg else v
    def skip(x, y):
        return (logx and x <= 0) or (logy and y <= 0) or not math.isfinite(y)
    xmin, xmax, ymin, ymax = 1e300, -1e300, 1e300, -1e300
    for _, xs, ys in series:
        for x, y in zip(xs, ys):
            if skip(x, y):
                continue
            xmin, xmax = min(xmin, ax(x, logx)), max(xmax, ax(x, logx))
            ymin, ymax = min(ymin, ax(y, logy)), max(ymax, ax(y, logy))
    if xmax <= xmin:
        xmax = xmin + 1
    if ymax <= ymin:
        ymax = ymin + 1
    def px(x):
        return ml + (ax(x, logx) - xmin) / (xmax - xmin) * (width - ml - mr)
    def py(y):
        return height - mb - (ax(y, logy) - ymin) / (ymax - ymin) * (height - mt - mb)
    g = "{:g}".format
    colors = ["#1f77b4", "#d62728", "#2ca02c", "#9467bd", "#ff7f0e", "#8c564b", "#17becf", "#7f7f7f"]
    o = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{width}" height="{height}">\n'
         '<rect width="100%" height="100%" fill="white"/>\n',
         f'<text x="{width // 2}" y="20" text-anchor="middle" font-size="15">{title}</text>\n',
         f'<text x="{width // 2}" y="{height - 12}" text-anchor="middle" font-size="12">{xlabel}</text>\n',
         f'<text x="16" y="{height // 2}" text-anchor="middle" font-size="12" transform="rotate(-90 16 '
         f'{height // 2})">{ylabel}</text>\n',
         f'<rect x="{ml}" y="{mt}" width="{width - ml - mr}" height="{height - mt - mb}" fill="none" '
         'stroke="black"/>\n']
    for k in range(5):
        fx, fy = xmin + (xmax - xmin) * k / 4.0, ymin + (ymax - ymin) * k / 4.0
        gx, gy = ml + (width - ml - mr) * k / 4.0, height - mb - (height - mt - mb) * k / 4.0
        lx, ly = "%.3g" % (10 ** fx if logx else fx), "%.3g" % (10 ** fy if logy else fy)
        o.append(f'<text x="{g(gx)}" y="{height - mb + 16}" text-anchor="middle" font-size="10">{lx}</text>\n')
        o.append(f'<text x="{ml - 6}" y="{g(gy + 3)}" text-anchor="end" font-size="10">{ly}</text>\n')
    for ci, (label, xs, ys) in enumerate(series):
        color = colors[ci % 8]
        pts = "".join(f"{g(px(x))},{g(py(y))} " for x, y in zip(xs, ys) if not skip(x, y))
        o.append(f'<polyline fill="none" stroke="{color}" stroke-width="1.5" points="{pts}"/>\n')
        o.append(f'<text x="{width - mr + 10}" y="{mt + 14 + 16 * ci}" font-size="11" fill="{color}">{label}</text>\n')
    o.append("</svg>\n")
    return "".join(o)


def write_sg_outputs(out_dir, hist: SgHistory, nx, ny, dt, snapshot_times=(), kle=None, pce=None, manifest=None):
    """The `solve-sg` output set (driver_solve_sg, experiments.cpp:393-449, and
    run_driver's manifest, :741-754), values in %.17g like CsvWriter
    (io.cpp:15-44), in the reference's output order:
      probe_<k>.csv     t,mean,std,u0..uP       (needs hist.probe_coeffs)
      kle_spectrum.csv  n,lambda                (kle = (sigma, bx, by, n_vars))
      pce_indices.csv   term,total_order,exponents (pce = (n_vars, p_out))
      iterations.csv    step,iterations,final_residual
      snapshot_<k>.csv  node_id,x,y,mean,std    (needs hist.full_state)
      probes.svg        probe mean / std lines  (write_svg_lines)
      manifest.json     command, config, seed, wall_seconds, version, outputs
                        (manifest = {"command", "config", "seed", "wall_seconds"})
    Every .csv is a pure function of the history: reruns are byte-identical
    (acceptance criterion 16).  Returns the written file names."""
    os.makedirs(out_dir, exist_ok=True)
    names = []

    def emit(name, text):
        with open(os.path.join(out_dir, name), "w", newline="") as f:
            f.write(text)
        names.append(name)

    pc = hist.probe_coeffs
    nt = 0 if pc is None or pc.size == 0 else pc.shape[1]
    for p in range(hist.probe_mean.shape[0]):
        header = "t,mean,std" + "".join(f",u{j}" for j in range(nt))
        rows = [[hist.times[s], hist.probe_mean[p, s], hist.probe_std[p, s]] + [pc[p, j, s] for j in range(nt)]
                for s in range(len(hist.times))]
        names.append(f"probe_{p}.csv")
        _write_csv(os.path.join(out_dir, names[-1]), header, rows)
    if kle is not None:
        emit("kle_spectrum.csv", kle_spectrum_csv(kle_spectrum(*kle)))
    if pce is not None:
        emit("pce_indices.csv", pce_indices_csv(pce_indices(*pce)))
    if len(hist.iterations):
        _write_csv(os.path.join(out_dir, "iterations.csv"), "step,iterations,final_residual",
                   [[s + 1, int(hist.iterations[s]), hist.residual[s]] for s in range(len(hist.iterations))])
        names.append("iterations.csv")
    if len(snapshot_times) and hist.full_state is not None:
        n = (nx - 1) * (ny - 1)
        nodes = (nx + 1) * (ny + 1)
        gi, gj = np.arange(nodes) % (nx + 1), np.arange(nodes) // (nx + 1)
        interior = (gi > 0) & (gi < nx) & (gj > 0) & (gj < ny)
        dof = np.where(interior, (gj - 1) * (nx - 1) + gi - 1, -1)
        for k, ts in enumerate(snapshot_times):
            step = min(len(hist.full_state) - 1, int(np.floor(ts / dt + 0.5)))  # std::llround
            mean, sd = moments(hist.full_state[step], n)
            mean_n = np.where(interior, mean[np.maximum(dof, 0)], 0.0)
            sd_n = np.where(interior, sd[np.maximum(dof, 0)], 0.0)
            rows = [[i, gi[i] / nx, gj[i] / ny, mean_n[i], sd_n[i]] for i in range(nodes)]
            names.append(f"snapshot_{k}.csv")
            _write_csv(os.path.join(out_dir, names[-1]), "node_id,x,y,mean,std", rows)
    if hist.probe_mean.shape[0]:
        series = []
        for p in range(hist.probe_mean.shape[0]):
            series.append((f"mean p{p}", hist.times, hist.probe_mean[p]))
            series.append((f"std p{p}", hist.times, hist.probe_std[p]))
        emit("probes.svg", svg_lines("SG pressure statistics", "t (s)", "pressure", series))
    if manifest is not None:
        import json
        m = {"command": manifest.get("command", "solve-sg"), "config": manifest.get("config", {}),
             "seed": manifest.get("seed", 0), "wall_seconds": manifest.get("wall_seconds", 0.0),
             "version": "0.1.0", "outputs": list(names)}
        emit("manifest.json", json.dumps(m, indent=2, sort_keys=True) + "\n")  # nlohmann::json dump(2)
    return names


class SchurSystem:
    """View of the device-resident interface system (include/sgwave/dd.hpp:71-96)."""

    def __init__(self, solver):
        self._s = solver

    @property
    def n_global(self):
        return self._s.n_global

    @property
    def n_corner(self):
        return self._s.n_corner * self._s.n_terms

    def matvec(self, x):
        x = _f64(x)
        y = np.zeros(self._s.n_global)
        _check(load_library().sgw_schur_matvec(self._s._h, _p(x), _p(y)))
        return y

    def apply_nn2(self, r):
        r = _f64(r)
        z = np.zeros(self._s.n_global)
        _check(load_library().sgw_apply_nn2(self._s._h, _p(r), _p(z)))
        return z

    def apply_nn1(self, r):
        """SchurSystem::apply_nn1 (src/dd.cpp:178-195); the solver must use precond "nn1"."""
        return self.apply_precond("nn1", r)

    def apply_lumped(self, r):
        """SchurSystem::apply_lumped (src/dd.cpp:159-176); the solver must use precond "lumped"."""
        return self.apply_precond("lumped", r)

    def apply_precond(self, kind, r):
        """make_preconditioner(system, kind)(r) (src/dd.cpp)."""
        r = _f64(r)
        z = np.zeros(self._s.n_global)
        _check(load_library().sgw_apply_precond(self._s._h, precond_from_string(kind), _p(r), _p(z)))
        return z

    def local_block(self, sub, which="S"):
        """Dense copy of subdomain `sub`'s local operator (verification hook):
        "S" = S_s, "Q" = S_rr^-1, "Psi" = S_rr^-1 S_rc; returns (matrix, gmap)."""
        w = {"S": 0, "Q": 1, "Psi": 2}[which]
        d = np.zeros(3, np.int64)
        L = load_library()
        _check(L.sgw_local_block(self._s._h, sub, w, None, None, _p(d)))
        a, r, c = (int(v) for v in d)
        rows, cols = {0: (a, a), 1: (r, r), 2: (r, c)}[w]
        out = np.zeros(rows * cols)
        g = np.zeros(a, np.int64)
        _check(L.sgw_local_block(self._s._h, sub, w, _p(out), _p(g), None))
        return out.reshape(cols, rows).T.copy(), g

    def coarse_operator(self):
        n = self.n_corner
        out = np.zeros(n * n)
        _check(load_library().sgw_coarse_operator(self._s._h, _p(out)))
        return out.reshape(n, n).T.copy()


PRECONDS = ("nn2", "nn1", "lumped")


class _LocalSchurC(C.Structure):  # sgw_local_schur
    _fields_ = [("n", C.c_int), ("S", C.c_void_p), ("gmap", C.c_void_p), ("weights", C.c_void_p),
                ("nr", C.c_int), ("r_idx", C.c_void_p), ("nc", C.c_int), ("c_idx", C.c_void_p),
                ("corner_gmap", C.c_void_p)]


@dataclass
class LocalSchur:
    """include/sgwave/dd.hpp:50-62: a subdomain's dense local Schur complement S
    (n x n), local -> global flat interface map, weights D_s, the remaining
    (r_idx) and corner (c_idx) local indices and the corners' global indices."""
    S: np.ndarray
    gmap: np.ndarray
    weights: np.ndarray
    r_idx: np.ndarray
    c_idx: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    corner_gmap: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))


class SchurFromLocals:
    """SchurSystem{n_global, n_corner, locals} with finalize() done on the GPU
    (src/dd.cpp:98-140), built from hand-made LocalSchur data as
    test_dd.cpp:123-151 does: matvec, apply_nn2, coarse_operator, pcg."""

    def __init__(self, n_global, n_corner, locals_):
        self.n_global, self.n_corner = int(n_global), int(n_corner)
        self._keep = []
        arr = (_LocalSchurC * max(1, len(locals_)))()
        for s, ls in enumerate(locals_):
            n = int(np.asarray(ls.gmap).size)
            S = np.asfortranarray(np.asarray(ls.S, np.float64).reshape(n, n))
            gm = np.ascontiguousarray(ls.gmap, np.int64)
            w = np.ascontiguousarray(ls.weights, np.float64)
            ri = np.ascontiguousarray(ls.r_idx, np.int32)
            ci = np.ascontiguousarray(ls.c_idx, np.int32)
            cg = np.ascontiguousarray(ls.corner_gmap, np.int64)
            self._keep += [S, gm, w, ri, ci, cg]
            arr[s] = _LocalSchurC(n, S.ctypes.data, gm.ctypes.data, w.ctypes.data, ri.size, ri.ctypes.data,
                                  ci.size, ci.ctypes.data, cg.ctypes.data)
        self._h = C.c_void_p()
        _check(load_library().sgw_schur_from_locals(self.n_global, self.n_corner, len(locals_), arr,
                                                    C.byref(self._h)))
        self._keep = []

    def __del__(self):
        if getattr(self, "_h", None):
            load_library().sgw_schur_free(self._h)
            self._h = None

    def _apply(self, fn, x):
        x = _f64(x)
        y = np.zeros(self.n_global)
        _check(fn(self._h, _p(x), _p(y)))
        return y

    def matvec(self, x):
        return self._apply(load_library().sgw_gschur_matvec, x)

    def apply_nn2(self, r):
        return self._apply(load_library().sgw_gschur_apply_nn2, r)

    def coarse_operator(self):
        F = np.zeros((self.n_corner, self.n_corner), order="F")
        _check(load_library().sgw_gschur_coarse_operator(self._h, _p(F)))
        return np.asarray(F)

    def pcg(self, rhs, tol=1e-10, max_iter=500):
        rhs = _f64(rhs)
        x = np.zeros(self.n_global)
        it, conv, hl = C.c_int(), C.c_int(), C.c_int()
        hist = np.zeros(max_iter + 2)
        _check(load_library().sgw_gschur_pcg(self._h, _p(rhs), tol, max_iter, _p(x), C.byref(it), C.byref(conv),
                                             _p(hist), hist.size, C.byref(hl)))
        return x, {"iterations": it.value, "converged": bool(conv.value), "residual_history": hist[:hl.value].copy()}


_HOST_OP = C.CFUNCTYPE(None, C.c_void_p, C.c_longlong, C.POINTER(C.c_double), C.POINTER(C.c_double))


def pcg(apply_op, apply_precond, rhs, tol, max_iter):
    """pcg(LinearOp, LinearOp, rhs, tol, max_iter) -> (x, PcgReport)
    (include/sgwave/pcg.hpp:15-21, src/pcg.cpp:7-50): the CG recurrence runs on
    the GPU (sgw_pcg_ops); apply_op / apply_precond are Python callables on
    numpy vectors (apply_precond None: identity)."""
    rhs = _f64(rhs)
    n = rhs.size
    err = []

    def wrap(f):
        def cb(_ctx, m, x, y):
            try:
                xv = np.ctypeslib.as_array(x, shape=(m,))
                np.ctypeslib.as_array(y, shape=(m,))[:] = np.asarray(f(xv.copy()), np.float64)
            except BaseException as e:  # noqa: BLE001 - re-raised after the call
                err.append(e)
                np.ctypeslib.as_array(y, shape=(m,))[:] = np.nan
        return _HOST_OP(cb)

    cop = wrap(apply_op)
    cpre = wrap(apply_precond) if apply_precond is not None else _HOST_OP()
    x = np.zeros(n)
    it, conv, hl = C.c_int(), C.c_int(), C.c_int()
    hist = np.zeros(max_iter + 2)
    rc = load_library().sgw_pcg_ops(n, cop, None, cpre, None, _p(rhs), tol, max_iter, _p(x), C.byref(it),
                                    C.byref(conv), _p(hist), hist.size, C.byref(hl))
    if err:
        raise err[0]
    _check(rc)
    return x, {"iterations": it.value, "converged": bool(conv.value), "residual_history": hist[:hl.value].copy()}


def precond_from_string(name) -> int:
    """precond_from_string (include/sgwave/dd.hpp:100): unknown names are rejected."""
    if name not in PRECONDS:
        raise SgInvalidArgument(SGW_EINVAL, f"unknown preconditioner {name!r}")
    return PRECONDS.index(name)


class ShardPlan:
    """Rank `rank`'s share of a `world`-rank decomposition (host.hpp Geometry,
    computed by libsgw_b200 on the host): the rx x ry rank grid, the owner of
    every subdomain, the rank's local interface nodes (global positions) and
    its halo (per peer, the shared local nodes in ascending global order)."""

    def __init__(self, nx, ny, px, py, world, rank):
        L = load_library()
        info = np.zeros(7, np.int64)
        _check(L.sgw_shard_plan(nx, ny, px, py, world, rank, _p(info), None, None, None, None, None))
        self.rx, self.ry, self.n_sub_owned, self.n_iface, n_peers, n_idx, self.n_iface_global = (int(v) for v in info)
        self.sub_owner = np.zeros(px * py, np.int32)
        self.iface_gpos = np.zeros(self.n_iface, np.int32)
        self.peers = np.zeros(n_peers, np.int32)
        self.peer_off = np.zeros(n_peers + 1, np.int32)
        self.peer_idx = np.zeros(n_idx, np.int32)
        _check(L.sgw_shard_plan(nx, ny, px, py, world, rank, _p(info), _p(self.sub_owner), _p(self.iface_gpos),
                                _p(self.peers), _p(self.peer_off), _p(self.peer_idx)))
        self.owned = np.flatnonzero(self.sub_owner == rank)

    def shared_with(self, i):
        """local interface nodes shared with peers[i]"""
        return self.peer_idx[self.peer_off[i]:self.peer_off[i + 1]]


def shard_plan(px: int, py: int, world_size: int, nx: int | None = None, ny: int | None = None) -> list[list[int]]:
    """Subdomains (row-major ids) owned by each rank: 2D blocks of the rx x ry
    rank grid with the shortest cut (host.hpp rank_grid)."""
    if not 1 <= world_size <= px * py:
        raise SgInvalidArgument(SGW_EINVAL, "need 1 <= world_size <= number of subdomains")
    owner = ShardPlan(nx or 8 * px, ny or 8 * py, px, py, world_size, 0).sub_owner
    return [list(np.flatnonzero(owner == r)) for r in range(world_size)]


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it, the caller broadcasts it)."""
    buf = C.create_string_buffer(128)
    _check(load_library().sgw_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return buf.raw


class LocalGroup:
    """W sharded solvers in one process on one device, each driven by its own
    thread (the exchange is host-synchronised; see include/sgw.h).  Every
    call is collective: use map() so all ranks make it concurrently."""

    def __init__(self, world_size):
        self.world_size = world_size
        self._g = C.c_void_p()
        _check(load_library().sgw_local_group_new(world_size, C.byref(self._g)))

    def map(self, fn, timeout=600.0):
        """[fn(rank) for rank in range(W)], each call on its own thread."""
        import threading
        out, err = [None] * self.world_size, []

        def body(r):
            try:
                out[r] = fn(r)
            except BaseException as e:  # noqa: BLE001 - re-raised below
                err.append(e)
                load_library().sgw_local_group_abort(self._g)  # the other ranks' collectives fail instead of hanging
        th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(self.world_size)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout)
        if any(t.is_alive() for t in th):
            raise SgError(SGW_ENCCL, "local group: a rank did not finish (collective mismatch?)")
        if err:
            raise err[0]
        return out

    def solvers(self, *args, **kw):
        return self.map(lambda r: SgSolver(*args, rank=r, world_size=self.world_size, local_group=self, **kw))

    def close(self):
        if getattr(self, "_g", None):
            load_library().sgw_local_group_free(self._g)
            self._g = None

    __del__ = close


class SgSolver:
    """B200 SgSolver (src/sg.cpp).  Setup (interior factorizations, local
    Schur complements, NN2 data) runs on the GPU in the constructor."""

    def __init__(self, nx, ny, px, py, coeff, tensor, density=1.0, alpha0=0.5445, alpha1=0.0174,
                 params: NewmarkParams | None = None, options: SgOptions | None = None, *, rank=0, world_size=1,
                 nccl_id: bytes | None = None, local_group: "LocalGroup | None" = None, solo: bool = False):
        """world_size > 1 shards the subdomains over ranks (include/sgw.h): one
        process per GPU with the rank-0 `nccl_id` (nccl_unique_id()), or, for
        tests on one device, one thread per rank sharing a LocalGroup."""
        L = load_library()
        self.params = params or NewmarkParams()
        self.options = options or SgOptions()
        self.nx, self.ny = nx, ny
        self._coeff = _f64(coeff)
        if self._coeff.ndim != 2 or self._coeff.shape[1] != (nx + 1) * (ny + 1):
            raise SgInvalidArgument(SGW_EINVAL, "coefficient field must be n_in x (nx+1)(ny+1)")
        ti = np.ascontiguousarray(tensor.i, np.int32)
        tj = np.ascontiguousarray(tensor.j, np.int32)
        tk = np.ascontiguousarray(tensor.k, np.int32)
        tv = _f64(tensor.v)
        prob = _Problem(nx, ny, px, py, self._coeff.shape[0], _p(self._coeff), int(tensor.n_output), len(tv),
                        _p(ti), _p(tj), _p(tk), _p(tv), density, alpha0, alpha1, self.params.gamma,
                        self.params.zeta, self.params.dt, self.options.tol, self.options.max_iter,
                        self.options.device, rank, world_size, None, precond_from_string(self.options.precond),
                        int(self.options.implicit_schur))
        if self._coeff.shape[0] != tensor.n_input:
            raise SgInvalidArgument(SGW_EINVAL, "SgSolver: coefficient terms do not match tensor input size")
        self.rank, self.world_size = rank, world_size
        h = C.c_void_p()
        if solo:  # rank `rank` of a world_size decomposition, constructed alone (sgw_create_solo)
            _check(L.sgw_create_solo(C.byref(prob), world_size, rank, C.byref(h)))
        elif local_group is not None:
            _check(L.sgw_create_local_group(C.byref(prob), world_size, rank, local_group._g, C.byref(h)))
        else:
            if world_size > 1 and (nccl_id is None or len(nccl_id) != 128):
                raise SgInvalidArgument(SGW_EINVAL, "world_size > 1 needs the 128-byte NCCL id of rank 0")
            if nccl_id is not None:
                self._nccl_id = C.create_string_buffer(bytes(nccl_id), 128)
                prob.nccl_id = C.cast(self._nccl_id, C.c_void_p)
            _check(L.sgw_create(C.byref(prob), C.byref(h)))
        self._h = h
        s = np.zeros(8, np.int64)
        _check(L.sgw_sizes(self._h, _p(s)))
        (self.n_dofs, self.n_terms, self.n_iface, self.n_corner, self.n_global, self.n_sub, _,
         self.device_bytes) = (int(v) for v in s)

    def close(self):
        if getattr(self, "_h", None):
            load_library().sgw_destroy(self._h)
            self._h = None

    __del__ = close

    def schur(self):
        return SchurSystem(self)

    def uses_direct(self):
        return False

    def set_stream(self, stream_handle: int):
        _check(load_library().sgw_set_stream(self._h, C.c_void_p(stream_handle)))

    def _apply(self, op, x):
        x = _f64(x)
        y = np.zeros_like(x)
        _check(load_library().sgw_apply_block(self._h, op, _p(x), _p(y)))
        return y

    def apply_block_mass(self, x):
        return self._apply(0, x)

    def apply_block_stiffness(self, x):
        return self._apply(1, x)

    def apply_block_transient(self, x):
        return self._apply(2, x)

    def pcg(self, rhs):
        rhs = _f64(rhs)
        x = np.zeros(self.n_global)
        it, conv = C.c_int(), C.c_int()
        cap = self.options.max_iter + 2
        hist = np.zeros(cap)
        _check(load_library().sgw_pcg(self._h, _p(rhs), _p(x), C.byref(it), C.byref(conv), _p(hist), cap))
        return x, {"iterations": it.value, "converged": bool(conv.value),
                   "residual_history": hist[hist >= 0].copy()}

    def run(self, u0_nodal, v0_nodal, n_steps, force: ForceSpec | None = None) -> SgHistory:
        u0, v0 = _f64(u0_nodal), _f64(v0_nodal)
        probes = np.ascontiguousarray(self.options.probe_nodes, np.int32)
        its = np.zeros(n_steps, np.int32)
        res = np.zeros(n_steps)
        pm = np.zeros((len(probes), n_steps + 1))
        ps = np.zeros_like(pm)
        pc = np.zeros((len(probes), self.n_terms, n_steps + 1))
        full = np.zeros((n_steps + 1, self.n_terms * self.n_dofs)) if self.options.store_full else None
        hist = _History(_p(its), _p(res), len(probes), _p(probes), _p(pm), _p(ps), _p(full), _p(pc))
        if force is not None and force.table is not None:
            # the C ABI reads (n_steps + 1) x n_nodes doubles straight from the caller's buffer
            tb = np.asarray(force.table)
            if tb.ndim != 2 or tb.shape[0] < n_steps + 1 or tb.shape[1] != u0.size:
                raise SgInvalidArgument(SGW_EINVAL, "force table must be (n_steps + 1) x n_nodes")
        f = (force or ForceSpec())._c()
        _check(load_library().sgw_run(self._h, _p(u0), _p(v0), n_steps, C.byref(f), C.byref(hist)))
        times = np.cumsum(np.r_[0.0, np.full(n_steps, self.params.dt)])
        return SgHistory(times, its, res, pm, ps, full, pc)

    # device-resident stepping (benchmarks)
    def init_state(self, u0_nodal, v0_nodal, force: ForceSpec | None = None):
        u0, v0 = _f64(u0_nodal), _f64(v0_nodal)
        f = (force or ForceSpec())._c()
        _check(load_library().sgw_init_state(self._h, _p(u0), _p(v0), C.byref(f)))

    def advance(self, n_steps):
        its = np.zeros(max(n_steps, 1), np.int32)
        _check(load_library().sgw_advance(self._h, n_steps, _p(its)))
        return its[:n_steps]

    def state(self):
        u = np.zeros(self.n_terms * self.n_dofs)
        _check(load_library().sgw_get_state(self._h, _p(u)))
        return u

    def stats(self):
        o = np.zeros(10)
        _check(load_library().sgw_stats(self._h, _p(o)))
        keys = ["setup_s", "pcg_ms", "step_ms", "iterations", "launches", "steps", "rhs_ms", "rec_ms",
                "matvecs", "nn2s"]
        return dict(zip(keys, o.tolist()))

    def reset_stats(self):
        _check(load_library().sgw_reset_stats(self._h))

    KERNEL_CLASSES = ("symv_S", "symv_Q", "interior_sweep", "sg_operator")

    def kernel_profile(self, enable=True):
        """Per-kernel-class device timings: {class: (total_ms, launches, algorithmic bytes/launch)}."""
        o = np.zeros(22)
        _check(load_library().sgw_kernel_profile(self._h, int(enable), _p(o)))
        out = {c: (o[3 * i], int(o[3 * i + 1]), o[3 * i + 2]) for i, c in enumerate(self.KERNEL_CLASSES)}
        out["bytes_per_pcg_iteration"] = o[12]
        names = ["S_tiles", "S_scatter", "update", "Q_tiles_psi", "coarse_assemble", "coarse_solve", "z_scatter",
                 "init_true_residual"]
        out["pcg_phases_ms"] = dict(zip(names, o[13:21].tolist()))
        out["sg_operator_flops"] = o[21]
        return out

    def bench_kernel(self, which, reps=20):
        """Average device ms of one Schur matvec (0), NN2 apply (1), SG-operator apply (2) or the
        step's SG-operator form with the mass term of a second input (3)."""
        o = np.zeros(1)
        _check(load_library().sgw_bench_kernel(self._h, which, reps, _p(o)))
        return float(o[0])


# ----------------------------------------------------- deterministic solver --
@dataclass
class SolveOptions:  # include/sgwave/det_loop.hpp:14-21
    precond: str = "nn2"
    tol: float = 1e-8
    max_iter: int = 500
    store_full: bool = False
    probe_nodes: list = field(default_factory=list)
    device: int = 0


@dataclass
class TimeHistory:  # include/sgwave/det_loop.hpp:23-30
    times: np.ndarray
    probe_u: np.ndarray                 # n_probes x (n_steps + 1)
    full_u: np.ndarray | None           # (n_steps + 1) x n_dofs
    iterations: np.ndarray              # PcgReport::iterations per step
    residual: np.ndarray

    def mean_iterations(self):          # det_loop.cpp:10-15
        return float(self.iterations.mean()) if len(self.iterations) else 0.0


class DetSolver:
    """DetSolver (include/sgwave/det_loop.hpp:37-52, src/det_loop.cpp) on the
    B200 path: the deterministic problem is the SG system with one chaos term
    (c_000 = 1, the coefficient field = speed_sq; test_sg.cpp:158-178), solved
    by the same kernels with the lumped / NN1 / NN2 preconditioner.  The
    preconditioner's local operators are built at construction, so
    set_preconditioner() rebuilds the GPU solver (setup is seconds at these
    sizes)."""

    def __init__(self, nx, ny, px, py, speed_sq, density=1.0, alpha0=0.5445, alpha1=0.0174,
                 params: NewmarkParams | None = None, options: SolveOptions | None = None):
        self.nx, self.ny, self.px, self.py = nx, ny, px, py
        self.speed_sq = _f64(speed_sq).reshape(1, -1)
        self.density, self.alpha0, self.alpha1 = density, alpha0, alpha1
        self.params = params or NewmarkParams()
        self.options = options or SolveOptions()
        self._build()

    def _build(self):
        o = self.options
        self._sg = SgSolver(self.nx, self.ny, self.px, self.py, self.speed_sq, triple_products(1, 0, 0),
                            self.density, self.alpha0, self.alpha1, self.params,
                            SgOptions(precond=o.precond, tol=o.tol, max_iter=o.max_iter, store_full=o.store_full,
                                      probe_nodes=list(o.probe_nodes), device=o.device))
        self.n_dofs = self._sg.n_dofs

    def schur(self):
        return self._sg.schur()

    def uses_direct(self):
        return False

    def set_preconditioner(self, kind):  # det_loop.hpp:50
        precond_from_string(kind)
        if kind != self.options.precond:
            self.options.precond = kind
            self._sg.close()
            self._build()

    def set_tolerance(self, tol):  # det_loop.hpp:51
        if tol != self.options.tol:
            self.options.tol = tol
            self._sg.close()
            self._build()

    def run(self, u0_nodal, v0_nodal, n_steps, force: ForceSpec | None = None) -> TimeHistory:
        h = self._sg.run(u0_nodal, v0_nodal, n_steps, force)
        probe_u = h.probe_coeffs[:, 0, :] if h.probe_coeffs is not None else h.probe_mean
        return TimeHistory(h.times, probe_u, h.full_state, h.iterations, h.residual)


def run_precond_comparison(nx, dt, t_final, partitions, tol=1e-8, max_iter=500, device=0):
    """run_precond_comparison (src/experiments.cpp:82-111): mean PCG iterations
    of the Gaussian-pulse problem per preconditioner and partition."""
    u0 = gaussian_pulse(nx, nx, 0.7, 0.7, 1.0, 0.01)
    v0 = np.zeros_like(u0)
    steps = int(math.ceil(t_final / dt - 1e-12))
    out = {"subdomain_counts": [], "lumped": [], "nn1": [], "nn2": []}
    for px, py in partitions:
        out["subdomain_counts"].append(px * py)
        for kind in ("lumped", "nn1", "nn2"):
            s = DetSolver(nx, nx, px, py, np.ones((nx + 1) ** 2), 1.0, 0.5445, 0.0174, NewmarkParams(dt=dt),
                          SolveOptions(precond=kind, tol=tol, max_iter=max_iter, device=device))
            out[kind].append(s.run(u0, v0, steps).mean_iterations())
            s._sg.close()
    return out
