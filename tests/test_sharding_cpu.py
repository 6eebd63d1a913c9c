"""Multi-rank decomposition of the hot path on CPU with gloo (world 2 and 4).

The sharded GPU solver (include/sgw.h, csrc/comm.hpp, csrc/shard.cu) gives
each rank a 2D block of subdomains and the interface nodes they touch, laid
out by libsgw_b200's own host code (sgw_shard_plan: the rank grid, the local
interface numbering and the halo lists).  The reference's subdomain sums become
  q = sum_s R_s^T S_s R_s p          (dd.cpp:142-157)   local partial + p2p halo
  z = sum_s R_s^T D_s zeta_s         (dd.cpp:230-250)   local partial + p2p halo
  d = sum_s B_s^T (f_c - Psi^T f_r)  (dd.cpp:214-226)   allreduce (coarse vector)
  F_cc                               (dd.cpp:128-137)   allreduce, once
and every interface dot counts each global node once (its lowest holder).
Here real processes run exactly that exchange pattern (gloo isend/irecv of
the shared partials, combined in ascending rank order like the device
halo_combine) on the oracle's local Schur complements, in the rank-local
numbering the library computes.  They must reproduce the oracle's unsharded
matvec, coarse operator, NN2 and PCG (pcg.cpp:7-50) iteration counts."""
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_2512_23027_b200.sgwave import ShardPlan, SgInvalidArgument, shard_plan

torch = pytest.importorskip("torch")
dist = pytest.importorskip("torch.distributed")
mp = pytest.importorskip("torch.multiprocessing")


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def pcg(matvec, precond, dot, b, tol, max_iter=500):
    """src/pcg.cpp:7-50 (x0 = 0; recurrence residual, then true-residual
    confirmation and restart from it without resetting p)."""
    x = np.zeros_like(b)
    bn = np.sqrt(dot(b, b))
    if bn == 0.0:
        return x, 0
    r = b.copy()
    z = precond(r)
    p = z.copy()
    rz = dot(r, z)
    for it in range(1, max_iter + 1):
        q = matvec(p)
        alpha = rz / dot(p, q)
        x += alpha * p
        r -= alpha * q
        if np.sqrt(dot(r, r)) / bn <= tol:
            rt = b - matvec(x)
            if np.sqrt(dot(rt, rt)) / bn <= tol:
                return x, it
            r = rt
        z = precond(r)
        rz_new = dot(r, z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    raise RuntimeError("pcg did not converge")


class ShardedSchur:
    """One rank's share of the SG interface problem in the library's local
    numbering, built from the oracle's local Schur complements."""

    def __init__(self, solver, plan: ShardPlan, rank, nt, allreduce):
        self.ar, self.plan, self.rank, self.nt = allreduce, plan, rank, nt
        nl, ng = plan.n_iface, plan.n_iface_global
        self.nl = nl
        self.n = nt * nl
        # local flat index j*nl + q <-> global flat j*ng + gpos[q]
        self.gidx = (np.arange(nt)[:, None] * ng + plan.iface_gpos[None, :]).ravel()
        g2l = {int(g): i for i, g in enumerate(self.gidx)}
        holders = [{rank} for _ in range(nl)]
        for i, peer in enumerate(plan.peers):
            for q in plan.shared_with(i):
                holders[q].add(int(peer))
        self.holders = holders
        own = np.array([min(h) == rank for h in holders], float)
        self.own = np.tile(own, nt)
        n_sub = len(plan.sub_owner)
        gm_all = [solver.local_schur(s)[1] for s in range(n_sub)]  # geometry: replicated, cheap
        cnt = np.zeros(solver.n_global)
        for g in gm_all:
            np.add.at(cnt, g, 1.0)
        wg = 1.0 / np.maximum(cnt, 1.0)  # D_s: 1 / multiplicity
        corners = np.flatnonzero(cnt == 4)
        self.nc = len(corners)
        cpos = np.full(solver.n_global, -1)
        cpos[corners] = np.arange(self.nc)
        self.subs = []
        fcc = np.zeros((self.nc, self.nc))
        for s in plan.owned:
            S, g = solver.local_schur(int(s))
            lg = np.array([g2l[int(v)] for v in g])
            c = cnt[g] == 4
            r = ~c
            Q = np.linalg.inv(S[np.ix_(r, r)])
            Psi = Q @ S[np.ix_(r, c)]
            F = S[np.ix_(c, c)] - S[np.ix_(r, c)].T @ Psi
            cp = cpos[g[c]]
            fcc[np.ix_(cp, cp)] += F
            self.subs.append((S, lg, wg[g], r, c, Q, Psi, cp))
        self.fcc = self.ar(fcc)  # the one-off exchange of the setup

    def halo(self, y):
        """complete a local partial: p2p exchange of the shared nodes' partials
        with every peer, each node summed over its holders in ascending rank"""
        plan = self.plan
        blocks, reqs = [], []
        for i, peer in enumerate(plan.peers):
            idx = plan.shared_with(i)
            send = torch.from_numpy(np.ascontiguousarray(y.reshape(self.nt, self.nl)[:, idx]).ravel())
            recv = torch.zeros_like(send)
            reqs += [dist.isend(send, int(peer)), dist.irecv(recv, int(peer))]
            blocks.append((send, recv, idx))
        for rq in reqs:
            rq.wait()
        part = {self.rank: y.reshape(self.nt, self.nl)}
        out = y.reshape(self.nt, self.nl).copy()
        got = {}
        for (send, recv, idx), peer in zip(blocks, plan.peers):
            rv = recv.numpy().reshape(self.nt, len(idx))
            for k, q in enumerate(idx):
                got[(int(peer), int(q))] = rv[:, k]
        for q in range(self.nl):
            h = sorted(self.holders[q])
            if len(h) < 2:
                continue
            acc = np.zeros(self.nt)
            for r in h:
                acc = acc + (part[r][:, q] if r == self.rank else got[(r, q)])
            out[:, q] = acc
        return out.ravel()

    def dot(self, a, b):
        return float(self.ar(np.array([np.sum(a * b * self.own)]))[0])

    def matvec(self, x):
        y = np.zeros(self.n)
        for S, lg, *_ in self.subs:
            np.add.at(y, lg, S @ x[lg])
        return self.halo(y)

    def apply_nn2(self, res):
        loc = []
        d = np.zeros(self.nc)
        for S, lg, w, r, c, Q, Psi, cp in self.subs:
            f = w * res[lg]
            fr, fc = f[r], f[c]
            np.add.at(d, cp, fc - Psi.T @ fr)
            loc.append((lg, w, r, c, Q, Psi, cp, fr))
        d = self.ar(d)
        uc = np.linalg.solve(self.fcc, d) if self.nc else d
        z = np.zeros(self.n)
        for lg, w, r, c, Q, Psi, cp, fr in loc:
            zeta = np.zeros(len(lg))
            zeta[r] = Q @ fr - Psi @ uc[cp]
            zeta[c] = uc[cp]
            np.add.at(z, lg, w * zeta)
        return self.halo(z)


CASES = {
    "16x16_4x2": (16, 16, 4, 2, 2, 2, 2),
    "ragged_14x10_4x3": (14, 10, 4, 3, 2, 3, 2),
    "strip_12x12_1x4": (12, 12, 1, 4, 2, 2, 2),  # no cross points: no coarse space
    "24x24_4x4": (24, 24, 4, 4, 2, 2, 2),
}


def _worker(rank, world, port, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def ar(a):
            t = torch.from_numpy(np.ascontiguousarray(a, np.float64).copy())
            dist.all_reduce(t)
            return t.numpy()

        nx, ny, px, py, L, pin, pout = CASES[case]
        coeff = O.lognormal_coeff(nx, ny, 0.3, 0.5, 0.5, L, pin)
        s = O.SgSolver(nx, ny, px, py, coeff, O.triple_products(L, pin, pout), dt=2e-3, tol=1e-10, threads=2)
        plan = ShardPlan(nx, ny, px, py, world, rank)
        sh = ShardedSchur(s, plan, rank, s.n_terms, ar)
        rng = np.random.default_rng(11)  # same vectors on every rank
        xg = rng.uniform(-1, 1, s.n_global)
        x = xg[sh.gidx]

        def rel(a, b):
            return np.linalg.norm(a - b) / np.linalg.norm(b)

        assert rel(sh.matvec(x), s.schur_matvec(xg)[sh.gidx]) <= 1e-12
        if sh.nc:
            assert rel(sh.fcc, s.coarse_operator()) <= 1e-12
        assert rel(sh.apply_nn2(x), s.apply_nn2(xg)[sh.gidx]) <= 1e-10
        bg = s.schur_matvec(xg)
        xs, its = pcg(sh.matvec, sh.apply_nn2, sh.dot, bg[sh.gidx], 1e-10)
        xr, itr = pcg(s.schur_matvec, s.apply_nn2, lambda a, b: float(a @ b), bg, 1e-10)
        assert abs(its - itr) <= 1, (its, itr)
        assert rel(xs, xr[sh.gidx]) <= 1e-8
        # every holder of a node holds the same value: the assembled global
        # solution (owned entries summed over ranks) reproduces each local copy
        xg_s = np.zeros(s.n_global)
        xg_s[sh.gidx] = xs * sh.own
        xg_s = ar(xg_s)
        assert np.array_equal(xg_s[sh.gidx], xs)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "16x16_4x2"), (2, "ragged_14x10_4x3"), (2, "strip_12x12_1x4"),
                                        (4, "24x24_4x4"), (4, "ragged_14x10_4x3")])
def test_gloo_decomposition_matches_oracle(world, case):
    mp.spawn(_worker, args=(world, free_port(), case), nprocs=world, join=True)


def test_shard_plan_covers_every_subdomain_once():
    for px, py in ((2, 1), (3, 1), (4, 2), (8, 8), (24, 24), (32, 32)):
        for world in (1, 2, 3, 4, 8):
            if world > px * py:
                with pytest.raises(SgInvalidArgument):
                    shard_plan(px, py, world)
                continue
            try:
                plan = shard_plan(px, py, world)
            except SgInvalidArgument:  # no rank grid rx x ry with rx <= px, ry <= py
                assert not any(world % a == 0 and a <= px and world // a <= py for a in range(1, world + 1))
                continue
            owned = sorted(s for r in plan for s in r)
            assert owned == list(range(px * py))
            sizes = [len(r) for r in plan]
            assert min(sizes) >= 1 and max(sizes) <= 2 * min(sizes)
            for r in plan:  # a 2D block: full rectangle of subdomains
                xs, ys = {s % px for s in r}, {s // px for s in r}
                assert len(r) == len(xs) * len(ys) and max(xs) - min(xs) + 1 == len(xs)


def test_rank_grid_and_halo_symmetry():
    # 8 ranks on 8x8 subdomains: a 4 x 2 grid; the halo lists of
    # two neighbours name the same global nodes in the same order
    nx, px, world = 64, 8, 8
    plans = [ShardPlan(nx, nx, px, px, world, r) for r in range(world)]
    assert (plans[0].rx, plans[0].ry) == (4, 2)
    for p in plans:
        assert p.n_iface_global == plans[0].n_iface_global
        assert np.all(np.diff(p.iface_gpos) > 0)
        for i, peer in enumerate(p.peers):
            q = plans[peer]
            k = list(q.peers).index(plans.index(p))
            assert np.array_equal(p.iface_gpos[p.shared_with(i)], q.iface_gpos[q.shared_with(k)])
    # the union of the local interfaces is the global interface
    allg = np.unique(np.concatenate([p.iface_gpos for p in plans]))
    assert np.array_equal(allg, np.arange(plans[0].n_iface_global))
    # interior rank of a 4x2 grid at C3 sizes: peers = horizontal, vertical and diagonal neighbours
    p = ShardPlan(512, 512, 16, 16, 8, 1)
    assert sorted(p.peers.tolist()) == [0, 2, 4, 5, 6]
