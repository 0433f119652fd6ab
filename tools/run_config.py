"""Run a BASELINE.json point configuration at full size on the GPU.

    python tools/run_config.py --config {1,2,3,5} [--steps 3] [--subsample 10000] [--scale 1.0]

Inputs follow SURVEY.md §8(d) (numpy default_rng; draws in the listed order).  Reports
device ms/step, (N+M)/s, phase times, and the relative l2 error on a random target
subsample against an fp64 direct sum over ALL sources, computed on the GPU with the
all-pairs drop-in kernel (fgt_gauss_direct_dev; minimum image for periodic, exact for
delta << 1/4).  Prints one JSON line.
"""

import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from tools.configs import CONFIGS  # noqa: E402
from tools.configs import generate as _generate  # noqa: E402


def generate(cfg_id, N):
    return _generate(cfg_id, N)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--subsample", type=int, default=10_000)
    ap.add_argument("--scale", type=float, default=1.0, help="N multiplier (debug)")
    ap.add_argument("--n-s", type=int, default=0, help="override s")
    args = ap.parse_args()
    import torch
    from paper_2305_07165_b200 import _lib, fgt_points_device
    from paper_2305_07165_b200.point_fgt import FgtParams

    cfg = dict(CONFIGS[args.config])
    N = int(cfg["N"] * args.scale)
    n_s = args.n_s or cfg["n_s"]
    t0 = time.perf_counter()
    y, q, x = generate(args.config, N)
    t_gen = time.perf_counter() - t0
    periodic = cfg["boundary"] == "periodic"
    prm = FgtParams(cfg["d"], cfg["delta"], cfg["eps"], n_s, periodic)
    dy, dq, dx = (torch.from_numpy(a).cuda() for a in (y, q, x))
    u = torch.empty(x.shape[0], dtype=torch.float64, device="cuda")
    ms, ph = [], None
    for i in range(args.steps + args.warmup):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _, ph = fgt_points_device(dy, dq, dx, cfg["delta"], cfg["eps"], n_s, cfg["boundary"],
                                  out=u, params=prm, return_times=True)
        b.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            ms.append(a.elapsed_time(b))
    # fp64 direct-sum spot check on a target subsample (all N sources)
    r = np.random.default_rng(123)
    sub = np.sort(r.choice(x.shape[0], size=min(args.subsample, x.shape[0]), replace=False))
    ds = torch.from_numpy(np.ascontiguousarray(x[sub])).cuda()
    ex = torch.zeros(sub.size, dtype=torch.float64, device="cuda")
    lib = _lib.load()
    t1 = time.perf_counter()
    _lib.check(lib.fgt_gauss_direct_dev(
        ctypes.c_void_p(ds.data_ptr()), sub.size, ctypes.c_void_p(dy.data_ptr()), N,
        ctypes.c_void_p(dq.data_ptr()), cfg["d"], 1.0 / cfg["delta"], float("inf"),
        1 if periodic else 0, ctypes.c_void_p(ex.data_ptr()), None))
    torch.cuda.synchronize()
    t_exact = time.perf_counter() - t1
    got = u.cpu().numpy()[sub]
    exn = ex.cpu().numpy()
    err = float(np.linalg.norm(got - exn) / np.linalg.norm(exn))
    out = {"config": args.config, "N": N, "M": int(x.shape[0]), "n_s": n_s, **cfg,
           "ms_per_step": float(np.mean(ms)), "points_per_s": (N + x.shape[0]) / (np.mean(ms) * 1e-3),
           "rel_l2_subsample": err, "bar_10eps": 10 * cfg["eps"], "pass": err <= 10 * cfg["eps"],
           "subsample": int(sub.size), "t_generate_s": t_gen, "t_exact_s": t_exact,
           "phases": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in ph.items()},
           "gpu_mem_peak_gb": torch.cuda.max_memory_allocated() / 1e9}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
