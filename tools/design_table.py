#!/usr/bin/env python
"""Rows of DESIGN.md's measurement table (section 8) from profiles/<tag>_bench_*.json.

  python tools/design_table.py r02d
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02d"


def load(name):
    p = os.path.join(ROOT, "profiles", f"{tag}_{name}.json")
    return json.load(open(p)) if os.path.exists(p) and os.path.getsize(p) else None


print("| Config | PCG GDOF·iter/s | ms / PCG iteration (frac of HBM) | ms / Newmark step | sweep frac | "
      "SG operator alone (frac) | e2e GDOF·iter/s | setup s |")
print("|---|---|---|---|---|---|---|---|")
for name, label in (("bench_C1", "C1"), ("bench_C2", "C2 (headline)"),
                    ("bench_C2_shard1", "C2, sharded code path on a 1-rank NCCL communicator"),
                    ("bench_C3", "C3"), ("bench_C5L8", "C5, L = 8")):
    d = load(name)
    if not d:
        continue
    pr, so = d["pcg_iteration_roofline"], d["kernels"].get("sg_operator_standalone")
    e2e = d.get("e2e") or {}
    sg = f"{so['ms_per_launch'] * 1e3:.1f} µs ({so['roofline_frac']:.2f})" if so else "—"
    print(f"| {label} | {d['value']:.3g} | {pr['ms_per_iteration']:.3g} ({pr['frac']:.2f}) | {d['ms_per_step']:.3g} | "
          f"{d['roofline']['frac']:.2f} | {sg} | {e2e.get('value', float('nan')):.3g} | {d['setup_s']:.1f} |")
w = [load("solo_C4_w4"), load("solo_C4_w8")]
if all(w):
    print("| C4, one rank of W = 4 / 8 (solo) | — | " + " / ".join(f"{x.get('ms_per_pcg_iteration', float('nan')):.3g}" for x in w) +
          " | — | — | — | — | " + " / ".join(f"{x.get('setup_s', float('nan')):.0f}" for x in w) + " |")
