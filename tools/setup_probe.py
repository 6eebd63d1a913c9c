import sys, time
sys.path.insert(0, '.')
import torch
import bench
import paper_2512_23027_b200 as sg
name = sys.argv[1]
c = bench.CONFIGS[name]
nx = c["nx"]
t0 = time.perf_counter()
coeff = sg.lognormal_coeff(nx, nx, c["sigma"], c["b"], c["b"], c["L"], c["p_in"])
t1 = time.perf_counter()
t = sg.triple_products(c["L"], c["p_in"], c["p_out"])
t2 = time.perf_counter()
s = sg.SgSolver(nx, nx, c["px"], c["px"], coeff, t, params=sg.NewmarkParams(dt=c["dt"]))
t3 = time.perf_counter()
print(f"{name}: coeff {t1-t0:.2f} s  tensor {t2-t1:.2f} s  SgSolver {t3-t2:.2f} s")
