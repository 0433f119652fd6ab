import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2305_07165_b200 import fgt_points
y, q, x = bench.gen_config2(10**6, 10**6)
hy, hq, hx = (torch.from_numpy(a).pin_memory().numpy() for a in (y, q, x))
for i in range(6):
    t0 = time.perf_counter()
    u, t = fgt_points(hy, hq, hx, 1e-4, 1e-9, 200, return_times=True)
    dt = time.perf_counter() - t0
    print(f"wall {dt*1e3:.2f} ms  h2d {t['h2d_ms']:.2f} total {t['total_ms']:.2f} d2h {t['d2h_ms']:.2f} form {t['form_ms']:.2f} tree {t['tree_ms']:.2f}")
from paper_2305_07165_b200.point_fgt import FgtParams
for i in range(3):
    t0 = time.perf_counter()
    FgtParams(3, 1e-4, 1e-9, 200, False, (0, 1))
    print(f"params {1e3*(time.perf_counter()-t0):.3f} ms")
