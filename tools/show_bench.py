#!/usr/bin/env python
"""Print the headline fields of every bench JSON line in the given log files."""
import json, sys
for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line.startswith('{'):
            if line.startswith('#'): print(line)
            continue
        d = json.loads(line)
        if 'roofline' not in d:
            print(f, line[:200]); continue
        k = d['kernels']['interior_sweep']
        print(f"{d['config']['workload'][:4]} value {d['value']:.3f} ms/step {d['ms_per_step']:.3f} sweep {k['ms_total']/k['launches']:.4f} ms frac {d['roofline']['frac']:.3f} "
              f"pcg-it {d['pcg_iteration_roofline']['ms_per_iteration']:.4f} ms frac {d['pcg_iteration_roofline']['frac']:.3f} bd {({a: round(b, 3) for a, b in d['step_breakdown_ms'].items()})}")
