"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the CPU oracle (oracle/*.cpp).

The oracle restates the reference sgwave SG-PCG/NN2 path on the CPU.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this module, and only as the checker or the CPU baseline —
never as the measured product path.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def build() -> str:
    """Compile the oracle with its own Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_lognormal_coeff.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                          C.c_double, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                          C.POINTER(C.c_int)]
        L.orc_local_maps.argtypes = [C.c_void_p, C.c_int] + [C.c_void_p] * 4 + [C.POINTER(C.c_longlong)] * 2
        L.orc_kle_lambdas.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, _dp]
        L.orc_triple_products.argtypes = [C.c_int] * 4 + [C.POINTER(C.c_int)] * 3 + [C.c_void_p] * 4
        L.orc_nearest_node.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double]
        L.orc_solver_create.argtypes = ([C.c_int] * 5 + [_dp, C.c_int, C.c_int, _ip, _ip, _ip, _dp]
                                        + [C.c_double] * 7 + [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)])
        L.orc_solver_destroy.argtypes = [C.c_void_p]
        L.orc_solver_sizes.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(dtype=np.int64)]
        L.orc_apply_block.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        L.orc_schur_apply.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        L.orc_coarse_operator.argtypes = [C.c_void_p, _dp]
        L.orc_local_schur.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_longlong)]
        L.orc_run.argtypes = [C.c_void_p, _dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_residual_history.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int]
        L.orc_timing.argtypes = [C.c_void_p, _dp]
        L.orc_local_blocks_create.argtypes = ([C.c_int] * 5 + [_dp, C.c_int, C.c_int, _ip, _ip, _ip, _dp]
                                              + [C.c_double] * 6 + [C.c_int, C.c_int,
                                                                    np.ctypeslib.ndpointer(dtype=np.int64),
                                                                    C.POINTER(C.c_void_p)])
        L.orc_local_blocks_get.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                           C.c_void_p]
        L.orc_pcg.argtypes = [C.c_void_p, _dp, _dp, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp, C.c_int, C.c_int,
                              C.c_double, C.c_int]
        L.orc_local_blocks_destroy.argtypes = [C.c_void_p]
        L.orc_single_block_nn2.argtypes = [C.c_int, _dp, _dp, _dp, C.c_double, C.POINTER(C.c_int)]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise RuntimeError(lib().orc_last_error().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------- inputs --
def mesh_coords(nx, ny):
    """Node coordinates of build_unit_square_mesh (src/mesh.cpp:15-58)."""
    i = np.tile(np.arange(nx + 1), ny + 1)
    j = np.repeat(np.arange(ny + 1), nx + 1)
    return i / nx, j / ny


def gaussian_pulse(nx, ny, x0=0.7, y0=0.7, beta=1.0, alpha=0.01):
    """src/experiments.cpp:14-22"""
    x, y = mesh_coords(nx, ny)
    return np.array([beta * math.exp(-((a - x0) ** 2 + (b - y0) ** 2) / alpha) for a, b in zip(x, y)])


def lognormal_coeff(nx, ny, sigma, bx, by, n_vars, p_in, g0=0.0):
    n_in = C.c_int()
    _check(lib().orc_lognormal_coeff(nx, ny, sigma, bx, by, g0, n_vars, p_in, None, 0, C.byref(n_in)))
    out = np.zeros((n_in.value, (nx + 1) * (ny + 1)))
    _check(lib().orc_lognormal_coeff(nx, ny, sigma, bx, by, g0, n_vars, p_in, _ptr(out), out.size,
                                     C.byref(n_in)))
    return out


def kle_lambdas(nx, ny, sigma, bx, by, n_modes):
    out = np.zeros(n_modes)
    _check(lib().orc_kle_lambdas(nx, ny, sigma, bx, by, n_modes, out))
    return out


class Tensor:
    """Sparse triple-product tensor, entries with j <= k (include/sgwave/pce.hpp:24-40)."""

    def __init__(self, n_input, n_output, i, j, k, v):
        self.n_input, self.n_output = n_input, n_output
        self.i, self.j, self.k, self.v = (np.ascontiguousarray(i, np.int32), np.ascontiguousarray(j, np.int32),
                                          np.ascontiguousarray(k, np.int32), np.ascontiguousarray(v, np.float64))

    def dense(self):
        g = np.zeros((self.n_input, self.n_output, self.n_output))
        g[self.i, self.j, self.k] = self.v
        g[self.i, self.k, self.j] = self.v
        return g


def triple_products(n_vars, p_in, p_out, quadrature=False):
    ni, no, ne = C.c_int(), C.c_int(), C.c_int()
    L = lib()
    _check(L.orc_triple_products(n_vars, p_in, p_out, int(quadrature), C.byref(ni), C.byref(no), C.byref(ne),
                                 None, None, None, None))
    i = np.zeros(ne.value, np.int32)
    j = np.zeros_like(i)
    k = np.zeros_like(i)
    v = np.zeros(ne.value)
    _check(L.orc_triple_products(n_vars, p_in, p_out, int(quadrature), C.byref(ni), C.byref(no), C.byref(ne),
                                 _ptr(i), _ptr(j), _ptr(k), _ptr(v)))
    return Tensor(ni.value, no.value, i, j, k, v)


def nearest_node(nx, ny, x, y):
    return lib().orc_nearest_node(nx, ny, x, y)


def cfl_dt(nx, c0_max, sigma, cfl=0.65):
    """cfl_timestep(mesh.h, conservative_cmax(c0, sigma), cfl) (src/experiments.cpp:32-34,
    src/newmark.cpp:51-56)."""
    h = math.sqrt((1.0 / nx) ** 2 + (1.0 / nx) ** 2)
    return cfl * h / (math.sqrt(c0_max) * math.exp(3.0 * sigma))


# ----------------------------------------------------------------- solver --
# PrecondKind (include/sgwave/dd.hpp:98): the SG path always uses nn2 (src/sg.cpp:330);
# the deterministic DetSolver (det_loop.hpp:14) selects any of the three.
PRECONDS = {"nn2": 0, "nn1": 1, "lumped": 2}


class SgSolver:
    """Oracle SgSolver (src/sg.cpp).  Same constructor arguments as the
    reference, with the mesh/partition given by their structured sizes."""

    def __init__(self, nx, ny, px, py, coeff, tensor: Tensor, density=1.0, alpha0=0.5445, alpha1=0.0174,
                 dt=1e-3, gamma=0.5, zeta=0.25, tol=1e-8, max_iter=500, threads=None, precond="nn2"):
        self.nx, self.ny = nx, ny
        coeff = np.ascontiguousarray(coeff, np.float64)
        threads = threads or os.cpu_count() or 1
        h = C.c_void_p()
        _check(lib().orc_solver_create(nx, ny, px, py, coeff.shape[0], coeff, tensor.n_output, len(tensor.v),
                                       tensor.i, tensor.j, tensor.k, tensor.v, density, alpha0, alpha1, gamma,
                                       zeta, dt, tol, max_iter, threads, PRECONDS[precond], C.byref(h)))
        self._h = h
        self.tol = tol
        s = np.zeros(6, np.int64)
        lib().orc_solver_sizes(self._h, s)
        self.n_dofs, self.n_terms, self.n_iface, self.n_corner, self.n_global, direct = (int(v) for v in s)
        self.uses_direct = bool(direct)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_solver_destroy(self._h)
            self._h = None

    def apply_block(self, x, op="transient"):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros_like(x)
        _check(lib().orc_apply_block(self._h, {"mass": 0, "stiffness": 1, "transient": 2}[op], x, y))
        return y

    def schur_matvec(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.n_global)
        _check(lib().orc_schur_apply(self._h, 0, x, y))
        return y

    def apply_nn2(self, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros(self.n_global)
        _check(lib().orc_schur_apply(self._h, 1, r, z))
        return z

    def apply_nn1(self, r):
        """SchurSystem::apply_nn1 (src/dd.cpp:178-195); needs precond="nn1"."""
        return self._schur_apply(2, r)

    def apply_lumped(self, r):
        """SchurSystem::apply_lumped (src/dd.cpp:159-176); needs precond="lumped"."""
        return self._schur_apply(3, r)

    def apply_precond(self, kind, r):
        """make_preconditioner(system, kind) (src/dd.cpp) applied to r."""
        return self._schur_apply({"nn2": 1, "nn1": 2, "lumped": 3}[kind], r)

    def _schur_apply(self, which, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros(self.n_global)
        _check(lib().orc_schur_apply(self._h, which, r, z))
        return z

    def pcg(self, rhs, tol=None, max_iter=500, precond="nn2"):
        """pcg(matvec, precond, rhs, tol, max_iter) (src/pcg.cpp:7-50) -> (x, report dict)."""
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.zeros(self.n_global)
        it, cv = C.c_int(), C.c_int()
        hist = np.zeros(max_iter + 2)
        _check(lib().orc_pcg(self._h, rhs, x, C.byref(it), C.byref(cv), hist, len(hist), PRECONDS[precond],
                             self.tol if tol is None else tol, max_iter))
        h = hist[hist >= 0]
        return x, {"iterations": it.value, "converged": bool(cv.value), "residual_history": h}

    def coarse_operator(self):
        out = np.zeros(self.n_corner * self.n_terms * self.n_corner * self.n_terms)
        lib().orc_coarse_operator(self._h, out)
        n = self.n_corner * self.n_terms
        return out.reshape(n, n).T.copy()

    def local_schur(self, s):
        a = C.c_longlong()
        lib().orc_local_schur(self._h, s, None, None, C.byref(a))
        S = np.zeros(a.value * a.value)
        g = np.zeros(a.value, np.int64)
        lib().orc_local_schur(self._h, s, _ptr(S), _ptr(g), C.byref(a))
        return S.reshape(a.value, a.value).T.copy(), g

    def local_schur_full(self, s):
        """LocalSchur s (dd.hpp:50-62): S, gmap, weights, r_idx, c_idx, corner_gmap"""
        S, g = self.local_schur(s)
        nr, nc = C.c_longlong(), C.c_longlong()
        lib().orc_local_maps(self._h, s, None, None, None, None, C.byref(nr), C.byref(nc))
        w = np.zeros(g.size)
        ri, ci = np.zeros(nr.value, np.int32), np.zeros(nc.value, np.int32)
        cg = np.zeros(nc.value, np.int64)
        lib().orc_local_maps(self._h, s, _ptr(w), _ptr(ri), _ptr(ci), _ptr(cg), C.byref(nr), C.byref(nc))
        return {"S": S, "gmap": g, "weights": w, "r_idx": ri, "c_idx": ci, "corner_gmap": cg}

    def run(self, u0, v0, n_steps, force_node=-1, f0=10.0, t0=0.1, amp=1.0, store_full=False, probes=()):
        u0 = np.ascontiguousarray(u0, np.float64)
        v0 = np.ascontiguousarray(v0, np.float64)
        iters = np.zeros(n_steps, np.int32)
        res = np.zeros(n_steps)
        N = self.n_terms * self.n_dofs
        full = np.zeros((n_steps + 1, N)) if store_full else None
        probes = np.ascontiguousarray(probes, np.int32)
        pm = np.zeros((len(probes), n_steps + 1))
        ps = np.zeros_like(pm)
        _check(lib().orc_run(self._h, u0, v0, n_steps, force_node, f0, t0, amp, _ptr(iters), _ptr(res),
                             _ptr(full), len(probes), _ptr(probes), _ptr(pm), _ptr(ps)))
        out = {"iterations": iters, "residual": res, "probe_mean": pm, "probe_std": ps}
        if store_full:
            out["full"] = full
        if not self.uses_direct:
            out["mean_iterations"] = float(iters.mean()) if n_steps else 0.0
        t = np.zeros(4)
        lib().orc_timing(self._h, t)
        out["t_setup"], out["t_pcg"], out["t_run"], out["total_iterations"] = t[0], t[1], t[2], int(t[3])
        return out

    def residual_history(self, k):
        buf = np.zeros(1024)
        n = lib().orc_residual_history(self._h, k, buf, len(buf))
        return buf[:n].copy()


class LocalBlocks:
    """One subdomain's S_s, S_rr^{-1} and Psi_s = S_rr^{-1} S_rc built alone
    (SgSolver::local_blocks, src/sg.cpp:186-246 + src/dd.cpp:112-120), for
    per-subdomain checks at sizes where the whole oracle exceeds host RAM."""

    def __init__(self, nx, ny, px, py, coeff, tensor: Tensor, s, density=1.0, alpha0=0.5445, alpha1=0.0174,
                 dt=1e-3, gamma=0.5, zeta=0.25, threads=None):
        coeff = np.ascontiguousarray(coeff, np.float64)
        sz = np.zeros(3, np.int64)
        h = C.c_void_p()
        _check(lib().orc_local_blocks_create(nx, ny, px, py, coeff.shape[0], coeff, tensor.n_output, len(tensor.v),
                                             tensor.i, tensor.j, tensor.k, tensor.v, density, alpha0, alpha1, gamma,
                                             zeta, dt, s, threads or os.cpu_count() or 1, sz, C.byref(h)))
        self._h = h
        self.a, self.r, self.c = (int(v) for v in sz)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_local_blocks_destroy(self._h)
            self._h = None

    def schur(self):
        S = np.zeros(self.a * self.a)
        g = np.zeros(self.a, np.int64)
        _check(lib().orc_local_blocks_get(self._h, _ptr(S), _ptr(g), None, 0, None, None))
        return S.reshape(self.a, self.a).T.copy(), g

    def srr_solve(self, V):
        """S_rr^{-1} V for V of shape (r, m)."""
        Vt = np.ascontiguousarray(np.asarray(V, np.float64).T)
        out = np.zeros_like(Vt)
        _check(lib().orc_local_blocks_get(self._h, None, None, _ptr(Vt), Vt.shape[0], _ptr(out), None))
        return out.T.copy()

    def psi(self):
        P = np.zeros(self.r * self.c)
        _check(lib().orc_local_blocks_get(self._h, None, None, None, 0, None, _ptr(P)))
        return P.reshape(self.c, self.r).T.copy()


def single_block_nn2(a, r, tol=1e-10):
    """test_dd.cpp:123-151: NN2 of a one-block, corner-free Schur system and the
    PCG iteration count it yields."""
    a = np.ascontiguousarray(np.asarray(a, np.float64).T)  # column-major
    r = np.ascontiguousarray(r, np.float64)
    z = np.zeros_like(r)
    it = C.c_int()
    _check(lib().orc_single_block_nn2(len(r), a, r, z, tol, C.byref(it)))
    return z, it.value
