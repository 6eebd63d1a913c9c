#!/usr/bin/env python
"""Benchmark of the per-Newmark-step SG-PCG / NN2 solve (BASELINE.json metric).

Ours:      python bench.py [--gpus N --steps K --warmup W]
Reference: python bench.py --impl reference ...   (CPU oracle restatement of the
           reference path on the host cores — the reference itself cannot be
           built here: Eigen3 + vendored doctest/CLI11/json are absent.)

A "step" is one Newmark step of configs[1] (C2): RHS + interior Dirichlet
solves + interface PCG with NN2 + recovery + update, on device-resident state.
`value` = PCG GDOF*iter/s = (P+1) N sum(iterations) / PCG device time / 1e9.
Prints one JSON line (rank 0).
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG GDOF·iter/s and s per Newmark step at (P+1)×N; % of HBM roofline"
UNIT = "GDOF·iter/s"

CONFIGS = {  # BASELINE.json configs
    "C1": dict(nx=64, px=4, L=2, p_in=4, p_out=2, sigma=0.3, b=0.5, dt=1e-3),
    "C2": dict(nx=256, px=8, L=3, p_in=6, p_out=3, sigma=0.3, b=0.5, dt=1e-3),
    "C3": dict(nx=512, px=16, L=4, p_in=6, p_out=3, sigma=0.4, b=0.3, dt=1e-3),
    # configs[3]: ~224 GB in the explicit formulation -> sharded over >= 2 GPUs (--gpus N)
    "C4": dict(nx=1024, px=32, L=6, p_in=4, p_out=2, sigma=0.3, b=0.5, dt=1e-3),
    # configs[4], the random-dimension sweep at p_in = 4; L = 12, 16 need >= 4 GPUs
    "C5L2": dict(nx=512, px=16, L=2, p_in=4, p_out=2, sigma=0.3, b=0.5, dt=1e-3),
    "C5L4": dict(nx=512, px=16, L=4, p_in=4, p_out=2, sigma=0.3, b=0.5, dt=1e-3),
    "C5L8": dict(nx=512, px=16, L=8, p_in=4, p_out=2, sigma=0.3, b=0.5, dt=1e-3),
}
ALPHA0, ALPHA1, TOL, F0, T0 = 0.5445, 0.0174, 1e-10, 10.0, 0.1


def workload_desc(name, c):
    nt = math.comb(c["L"] + c["p_out"], c["p_out"])
    return (f"{name}: {c['nx']}x{c['nx']} P1 grid ({(c['nx'] + 1) ** 2} nodes), {c['px']}x{c['px']} subdomains, "
            f"KL modes {c['L']}, P+1={nt}, p_in={c['p_in']}, sigma={c['sigma']}, corr.len={c['b']}, dt={c['dt']}, "
            f"Ricker f0={F0} Hz t0={T0} at (0.5,0.5), Newmark beta=1/4 gamma=1/2, "
            f"alpha0={ALPHA0} alpha1={ALPHA1}, PCG tol {TOL}, fp64")


# FP64 FMA peak measured on this pool's B200s (tools/bench_fp64.cu,
# profiles/r02_fp64_peak.txt: 16.77 TFMA/s with 32 warps/SM x 8 chains)
FP64_TFLOPS = 2 * 16.77


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        self.f = tempfile.NamedTemporaryFile("w+", delete=False, suffix=".csv")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        rows = [[x.strip() for x in r] for r in rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, nm in enumerate(names):
                if r[3 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def cpu_oracle_run(c, warmup, steps, threads):
    """Oracle (CPU restatement of the reference path): setup untimed, then
    `warmup` + `steps` Newmark steps; returns PCG GDOF*iter/s and s/step."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    nx = c["nx"]
    coeff = O.lognormal_coeff(nx, nx, c["sigma"], c["b"], c["b"], c["L"], c["p_in"])
    tensor = O.triple_products(c["L"], c["p_in"], c["p_out"])
    t0 = time.perf_counter()
    s = O.SgSolver(nx, nx, c["px"], c["px"], coeff, tensor, alpha0=ALPHA0, alpha1=ALPHA1, dt=c["dt"], tol=TOL,
                   threads=threads)
    setup = time.perf_counter() - t0
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    # warm-up steps then timed steps, one continuous trajectory
    out = s.run(z, z, warmup + steps, force_node=node, f0=F0, t0=T0) if warmup == 0 else None
    if out is None:
        w = s.run(z, z, warmup, force_node=node, f0=F0, t0=T0)
        t_w, pcg_w, it_w = w["t_run"], w["t_pcg"], w["total_iterations"]
        out = s.run(z, z, warmup + steps, force_node=node, f0=F0, t0=T0)
        t_run, t_pcg = out["t_run"] - t_w, out["t_pcg"] - pcg_w
        iters = out["total_iterations"] - it_w
    else:
        t_run, t_pcg, iters = out["t_run"], out["t_pcg"], out["total_iterations"]
    gdof = s.n_terms * (nx + 1) ** 2
    return {"value": gdof * iters / t_pcg / 1e9, "value_step": gdof * iters / t_run / 1e9, "s_per_step": t_run / steps,
            "iterations": iters, "setup_s": setup, "pcg_s": t_pcg, "n_terms": s.n_terms}


def run_reference(args, c, name):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    r = cpu_oracle_run(c, args.warmup, args.steps, threads)
    sample = (f"{name} full problem, setup excluded ({r['setup_s']:.1f} s), {args.warmup} warm-up + "
              f"{args.steps} timed Newmark steps, {threads} threads (std::thread over subdomains)")
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["s_per_step"] * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (deterministic KLE inputs; seeds have no effect on the SG solve)",
            "config": {"workload": workload_desc(name, c), "GDOF": r["n_terms"] * (c["nx"] + 1) ** 2 / 1e9},
            "s_per_newmark_step": r["s_per_step"], "pcg_iterations": r["iterations"],
            "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            # e2e: iterations over the WHOLE time-loop wall time (RHS, interior
            # solves, recovery included): the same definition as the GPU arm's e2e
            "e2e": {"value": r["value_step"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                    "note": "sum(iterations) (P+1) N / whole time-loop wall time (as the GPU arm's e2e)"},
            "note": "reference C++ needs Eigen3 and vendored doctest/CLI11/json (absent): oracle/ restatement timed"}
    print(json.dumps(line), flush=True)


def run_solo(args, c, name, sg):
    """One rank of a W-rank decomposition built alone on this GPU (sgw_create_solo):
    per-rank device memory, setup time and the shard's PCG iteration time
    (phase-split kernels, exchanges deliver zeros).  Unmeasured on hardware as
    a multi-GPU run: it times one shard's kernels, not the NVLink exchanges."""
    import torch

    nx = c["nx"]
    coeff = sg.lognormal_coeff(nx, nx, c["sigma"], c["b"], c["b"], c["L"], c["p_in"])
    tensor = sg.triple_products(c["L"], c["p_in"], c["p_out"])
    t0 = time.perf_counter()
    solver = sg.SgSolver(nx, nx, c["px"], c["px"], coeff, tensor, alpha0=ALPHA0, alpha1=ALPHA1,
                         params=sg.NewmarkParams(dt=c["dt"]),
                         options=sg.SgOptions(tol=1e-30, max_iter=args.steps), rank=args.solo_rank,
                         world_size=args.solo_world, solo=True)
    setup_s = time.perf_counter() - t0
    rhs = np.sin(0.001 * np.arange(solver.n_global) + 0.3)
    solver.pcg(rhs)  # warm-up (graph capture)
    solver.reset_stats()
    _, rep = solver.pcg(rhs)
    st = solver.stats()
    torch.cuda.synchronize()
    plan = sg.ShardPlan(nx, nx, c["px"], c["px"], args.solo_world, args.solo_rank)
    line = {"mode": "solo-rank loopback (one shard on one GPU; exchanges deliver zeros; not a multi-GPU measurement)",
            "config": {"workload": workload_desc(name, c), "world": args.solo_world, "rank": args.solo_rank,
                       "rank_grid": [plan.rx, plan.ry], "owned_subdomains": int(plan.n_sub_owned),
                       "local_interface_nodes": int(plan.n_iface), "halo_peers": plan.peers.tolist(),
                       "halo_doubles_per_exchange": int(len(plan.peer_idx)) * solver.n_terms},
            "device_bytes": solver.device_bytes, "setup_s": setup_s, "pcg_iterations": rep["iterations"],
            "ms_per_pcg_iteration": st["pcg_ms"] / max(rep["iterations"], 1)}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-steps", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--implicit-schur", action="store_true",
                    help="reduced-memory mode (S_s not stored, applied through the interior solve)")
    ap.add_argument("--force-shard", action="store_true",
                    help="test hook: the sharded code path (NCCL communicator) even on one rank")
    ap.add_argument("--solo-rank", type=int, default=None,
                    help="loopback: construct only this rank of a --solo-world decomposition on one GPU")
    ap.add_argument("--solo-world", type=int, default=2)
    ap.add_argument("--mode", default="shard", choices=["shard", "replica"],
                    help="N>1: shard the subdomains over the ranks (one problem, NCCL sums) or run N replicas")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    c = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, c, args.config)

    import torch
    import paper_2512_23027_b200 as sg

    if args.solo_rank is not None:
        return run_solo(args, c, args.config, sg)
    rank, world, local = dist_env()
    if world > 1 or args.force_shard:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    nx = c["nx"]
    coeff = sg.lognormal_coeff(nx, nx, c["sigma"], c["b"], c["b"], c["L"], c["p_in"])
    tensor = sg.triple_products(c["L"], c["p_in"], c["p_out"])
    node = sg.nearest_node(nx, nx, 0.5, 0.5)
    shard = (world > 1 and args.mode == "shard") or args.force_shard
    kw = {}
    if shard:  # rank r owns a 2D block of subdomains (sgw_shard_plan); the NCCL id travels over torch.distributed
        ids = [sg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        kw = dict(rank=rank, world_size=world, nccl_id=ids[0])
    t0 = time.perf_counter()
    solver = sg.SgSolver(nx, nx, c["px"], c["px"], coeff, tensor, alpha0=ALPHA0, alpha1=ALPHA1,
                         params=sg.NewmarkParams(dt=c["dt"]),
                         options=sg.SgOptions(tol=TOL, device=local, implicit_schur=args.implicit_schur), **kw)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    solver.set_stream(stream.cuda_stream)
    gdof = solver.n_terms * (nx + 1) ** 2
    z = np.zeros((nx + 1) ** 2)
    force = sg.ForceSpec(node=node, f0=F0, t0=T0)
    solver.init_state(z, z, force)
    solver.advance(args.warmup)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    torch.cuda.synchronize()
    barrier()
    solver.reset_stats()
    solver.kernel_profile(True)
    launches0 = solver.stats()["launches"]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.profiler.start()  # ncu --profile-from-start off: launch list of the timed region only
        ev0.record(stream)
        its = solver.advance(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    barrier()
    ms = ev0.elapsed_time(ev1)
    st = solver.stats()
    kp = solver.kernel_profile(False)
    launches = int(st["launches"] - launches0)
    pcg_ms, iters = st["pcg_ms"], int(its.sum())
    if world > 1:
        t = torch.tensor([ms, pcg_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        n = torch.tensor([float(iters)], device="cuda")
        torch.distributed.all_reduce(n)
        ms, pcg_ms, iters_all = float(t[0]), float(t[1]), int(n[0])
        if shard:  # one problem: every rank runs the same iterations
            iters_all = iters
    else:
        iters_all = iters
    value = gdof * iters_all / (pcg_ms / 1e3) / 1e9

    peak, peak_src = measured_peaks()
    # dominant kernel of the timed region
    classes = {k: v for k, v in kp.items() if isinstance(v, tuple) and v[1] > 0}
    dom = max(classes, key=lambda k: classes[k][0])
    dms, dn, dbytes = classes[dom]
    achieved = dbytes / (dms / dn / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            traffic = json.load(f).get(args.config, {}).get(dom, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    kernels = {k: {"ms_total": v[0], "launches": v[1], "algorithmic_bytes_per_launch": v[2],
                   "achieved_GBs": (v[2] / (v[0] / v[1] / 1e3) / 1e9) if v[1] else None}
               for k, v in classes.items()}
    # standalone fused SG-operator apply (apply_block_transient, K11), outside the timed region
    sgop_ms = solver.bench_kernel(2, reps=20)
    sgop_bytes, sgop_flops = kp["sg_operator"][2], kp["sg_operator_flops"]
    # roofline = max(bytes / HBM peak, flops / FP64 peak); the
    # 3-value stored-stencil form's bytes 8 n (3 n_in + 2 (P+1)) for reference
    n_dofs = (nx - 1) ** 2
    b3 = 8.0 * n_dofs * (3 * tensor.n_input + 2 * tensor.n_output)
    t_roof = max(sgop_bytes / (peak * 1e9), sgop_flops / (FP64_TFLOPS * 1e12))
    kernels["sg_operator_standalone"] = {
        "ms_per_launch": sgop_ms, "algorithmic_bytes_per_launch": sgop_bytes, "algorithmic_flops_per_launch": sgop_flops,
        "achieved_GBs": sgop_bytes / (sgop_ms / 1e3) / 1e9, "achieved_TFLOPs": sgop_flops / (sgop_ms / 1e3) / 1e12,
        "frac_of_peak": sgop_bytes / (sgop_ms / 1e3) / 1e9 / peak,
        "roofline_ms": t_roof * 1e3, "roofline_frac": t_roof / (sgop_ms / 1e3),
        "fp64_peak_TFLOPs": FP64_TFLOPS,
        "frac_vs_3value_stored_form": b3 / (sgop_ms / 1e3) / 1e9 / peak,
        "note": "2 stored couplings per node and term (sgop.cu); L2 flushed (read) before each launch"}
    b_iter = kp["bytes_per_pcg_iteration"]
    iter_ms = pcg_ms / max(iters, 1)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic KLE/PCE inputs of the config; seeds have no effect on the SG solve)",
        "config": {"workload": workload_desc(args.config, c), "GDOF": gdof / 1e9,
                   "parallelism": "single GPU" if world == 1 else (
                       f"{world} GPUs, 2D blocks of subdomains {[len(r) for r in sg.shard_plan(c['px'], c['px'], world)]}, "
                       "interface halo by ncclSend/ncclRecv, coarse vector + CG scalars by ncclAllReduce, "
                       "phase-split PCG in a CUDA graph (WHILE node)" if shard else f"{world} independent replicas"),
                   "l2": "inputs larger than L2: S+Q tiles stream ~2.7 GB per PCG iteration (L2 126 MB)",
                   **({"mode": "reduced-memory (implicit Schur: S_s applied through the interior sweep)"}
                      if args.implicit_schur else {})},
        "s_per_newmark_step": ms / args.steps / 1e3,
        "pcg_iterations": iters_all, "mean_iterations_per_step": iters / args.steps,
        "setup_s": setup_s,
        "roofline": {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src},
        "pcg_iteration_roofline": {"bytes_per_iteration": b_iter, "ms_per_iteration": iter_ms,
                                   "achieved": b_iter / (iter_ms / 1e3) / 1e9,
                                   "frac": b_iter / (iter_ms / 1e3) / 1e9 / peak},
        "kernels": kernels,
        "pcg_phases_ms_per_iteration": {k: v / max(iters, 1) for k, v in kp["pcg_phases_ms"].items()},
        # per Newmark step (CUDA events of the step): RHS (predictors, local force,
        # first interior sweep, g assembly), interface PCG, recovery (second
        # sweep) + update
        "step_breakdown_ms": {"rhs": st["rhs_ms"] / args.steps, "pcg": st["pcg_ms"] / args.steps,
                              "recovery_update": st["rec_ms"] / args.steps},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }

    if not args.no_e2e:
        # end to end through the public C ABI with host buffers: sgw_run with a
        # nodal force table (one row uploaded per step) and host-side history
        table = np.zeros((args.steps + 1, (nx + 1) ** 2))
        tt = 0.0
        for k in range(args.steps + 1):
            table[k, node] = sg.ricker(tt, F0, T0)
            tt += c["dt"]
        solver.options.probe_nodes = [node]
        solver.run(z, z, 2, sg.ForceSpec(table=table[:3].copy()))  # untimed warm-up of the API path
        torch.cuda.synchronize()
        barrier()
        w0 = time.perf_counter()
        h = solver.run(z, z, args.steps, sg.ForceSpec(table=table))
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        if world > 1:
            t = torch.tensor([wall], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            wall = float(t[0])
        e_iters = int(h.iterations.sum()) * (1 if shard else world)
        line["e2e"] = {"value": gdof * e_iters / wall / 1e9, "unit": UNIT,
                       "h2d_bytes_per_step": 8 * (nx + 1) ** 2 + 2 * 8 * (nx + 1) ** 2 / args.steps,
                       "d2h_bytes_per_step": 8 * (h.iterations.mean() + 2) + 16,
                       "wall_s": wall, "note": "sgw_run: u0/v0 + one nodal force row per step H2D; "
                                               "PCG residual scalars + probe history D2H"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        r = cpu_oracle_run(c, 1, args.cpu_steps, threads)
        line["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"{args.config} full problem, setup excluded ({r['setup_s']:.0f} s), "
                                          f"1 warm-up + {args.cpu_steps} timed Newmark steps, PCG time only",
                                "s_per_newmark_step": r["s_per_step"], "e2e_value": r["value_step"]}
        # per Newmark step, device-resident GPU step vs the oracle's whole step
        line["per_step_speedup_vs_cpu_baseline"] = r["s_per_step"] / (ms / args.steps / 1e3)
        if "e2e" in line:
            line["e2e"]["speedup_vs_cpu_baseline_e2e"] = line["e2e"]["value"] / r["value_step"]
    if rank == 0:
        print(json.dumps(line), flush=True)
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
