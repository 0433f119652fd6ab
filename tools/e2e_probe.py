"""Where the end-to-end (host API) time of config 2 goes, beyond H2D + device + D2H."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tools import configs  # noqa: E402
from paper_2305_07165_b200 import fgt_points, _lib
from paper_2305_07165_b200 import point_fgt as pf
y, q, x = configs.config2(10**6, 10**6)
hy, hq, hx = (torch.from_numpy(a).pin_memory().numpy() for a in (y, q, x))
for i in range(6):
    t0 = time.perf_counter()
    u, t = fgt_points(hy, hq, hx, 1e-4, 1e-9, 200, return_times=True)
    dt = time.perf_counter() - t0
    print(f"wall {dt*1e3:.2f} ms  h2d {t['h2d_ms']:.2f} total {t['total_ms']:.2f} d2h {t['d2h_ms']:.2f} "
          f"form {t['form_ms']:.2f} tree {t['tree_ms']:.2f}")
for i in range(3):
    c = [time.perf_counter()]
    src, qq, tgt, dim = pf._prep(hy, hq, hx, False); c.append(time.perf_counter())
    prm = pf.FgtParams(dim, 1e-4, 1e-9, 200, False, (0, 1)); c.append(time.perf_counter())
    uu = pf._host_out(tgt.shape[0]); c.append(time.perf_counter())
    times = _lib.FgtPhaseTimes(); P = _lib.ptr
    _lib.check(_lib.load().fgt_points(P(src), src.shape[0], P(qq), P(tgt), tgt.shape[0], ctypes.byref(prm.tp),
                                      ctypes.byref(prm.pw), P(uu), ctypes.byref(times)))
    c.append(time.perf_counter())
    d = times.as_dict()
    print("prep %.3f params %.3f out %.3f call %.3f | h2d+total+d2h %.3f" % tuple(
        [1e3 * (c[k + 1] - c[k]) for k in range(4)] + [d['h2d_ms'] + d['total_ms'] + d['d2h_ms']]))
