#!/usr/bin/env python
"""Markdown rows of BASELINE.md's results table from profiles/<tag>_bench_<config>.json.

  python tools/results_table.py r02b
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
NAMES = {"C1": "C1 64², 4×4, P+1=6", "C2": "C2 256², 8×8, P+1=20", "C3": "C3 512², 16×16, P+1=35",
         "C5L8": "C5 512², 16×16, L=8 (P+1=45)"}
PARITY = {"C1": "Δiters 0, 1e-12 (50 steps vs oracle)", "C2": "Δiters 0 (398 = 398), 1.3e-12 (100 steps vs oracle)",
          "C3": "per-subdomain S_s, S_rr⁻¹, Ψ_s vs oracle ≤ 1e-10; explicit / reduced-memory / 2-rank trajectories",
          "C5L8": "per-subdomain blocks vs oracle ≤ 1e-10"}
print("| Config | GPUs | Host cores | Mean iters/step (CPU / GPU) | PCG GDOF·iter/s CPU | PCG GDOF·iter/s GPU | s/step CPU | "
      "s/step GPU | PCG GB/s | % HBM (8 TB/s) | % HBM (measured) | SG-op GB/s (% HBM) | Parity (Δiters, rel L2) |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for c, name in NAMES.items():
    p = os.path.join(ROOT, "profiles", f"{tag}_bench_{c}.json")
    if not os.path.exists(p):
        continue
    d = json.load(open(p))
    cb = d.get("cpu_baseline") or {}
    pr = d["pcg_iteration_roofline"]
    so = d["kernels"].get("sg_operator_standalone", {})
    it = d["mean_iterations_per_step"]
    print(f"| {name} | 1 | {cb.get('cores', '—')} | {(str(it) + ' / ' + str(it)) if cb else '— / ' + str(it)} | "
          f"{cb.get('value', float('nan')):.4f} | {d['value']:.3f} | {cb.get('s_per_newmark_step', float('nan')):.4f} | "
          f"{d['s_per_newmark_step']:.5f} | {pr['achieved']:.0f} | {100 * pr['achieved'] / 8000:.0f} % | {100 * pr['frac']:.0f} % | "
          f"{so.get('achieved_GBs', float('nan')):.0f} ({100 * so.get('frac_of_peak', float('nan')):.0f} %) | {PARITY[c]} |")
