"""Per-rank cost of the strong-scaling shares, measured on ONE GPU.

    python tools/share_probe.py [--sizes 1,2,4,8] [--config 2|5] [--n N] [--mode exchange|recompute|sequential]

For each world size P it runs rank r's share (fgt_points_device(..., share=(r, P))) for
every r on the same GPU, one after another, and reports the per-rank CUDA-event step times.
The max over ranks is what a P-GPU run of bench.py would measure per step (each rank
rebuilds the replicated tree and lists, forms the expansions its targets need, and evaluates
its own targets; there is no data-path collective).  Inputs: BASELINE config 2 or 5
(tools/configs.py).  --mode sequential runs the exchange path one rank at a time with a
zero-filled halo of the right size (timing only: the ranks' values are not combined), so a
10^8-point config fits one GPU's memory.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from tools import configs  # noqa: E402
from paper_2305_07165_b200 import fgt_points_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1,2,4,8")
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 5])
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--mode", choices=["recompute", "exchange", "sequential"], default="exchange")
    a = ap.parse_args()
    cfg = configs.CONFIGS[a.config]
    a.n = a.n or cfg["N"]
    a.args = (cfg["delta"], cfg["eps"], cfg["n_s"], cfg["boundary"])
    y, q, x = configs.generate(a.config, a.n)
    dy, dq, dx = (torch.from_numpy(v).cuda() for v in (y, q, x))
    del y, q, x
    out = {}
    if a.mode == "exchange":
        return exchange_probe(a, dy, dq, dx)
    if a.mode == "sequential":
        return sequential_probe(a, dy, dq, dx)
    for P in (int(s) for s in a.sizes.split(",")):
        per = []
        for r in range(P):
            best = None
            for _ in range(a.reps):
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                _, t = fgt_points_device(dy, dq, dx, *a.args, return_times=True, share=(r, P))
                e.record()
                torch.cuda.synchronize()
                ms = s.elapsed_time(e)
                if best is None or ms < best[0]:
                    best = (ms, {k: round(t[k], 3) for k in ("tree_ms", "lists_ms", "form_ms", "gather_ms",
                                                            "eval_ms", "direct_ms")},
                            dict(n_spread_boxes=t["n_spread_boxes"], n_src_spread=t["n_src_spread"],
                                 n_psi=t["n_psi"], n_tgt_psi=t["n_tgt_psi"]))
            per.append({"rank": r, "ms": round(best[0], 3), **best[1], **best[2]})
        mx = max(p["ms"] for p in per)
        out[P] = {"max_rank_ms": mx, "points_per_s": 2 * a.n / (mx * 1e-3), "ranks": per}
        print(json.dumps({"P": P, "max_rank_ms": mx, "est_points_per_s": 2 * a.n / (mx * 1e-3),
                          "rank_ms": [p["ms"] for p in per],
                          "slowest": max(per, key=lambda p: p["ms"])}))
    return out


def exchange_probe(a, dy, dq, dx):
    """Owner-formed expansions + halo all-to-all: per rank, time begin (tree, lists, own
    expansions, pack) and finish (unpack, translation, evaluation, near field) with CUDA
    events; the all-to-all itself is emulated by device copies and reported as bytes (the
    NVLink time is bytes / ~400 GB/s per direction, NCCL all-to-all over NVSwitch)."""
    from paper_2305_07165_b200.point_fgt import fgt_points_exchange_begin
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
    from test_gpu_parity import _emulated_exchange
    for P in (int(s) for s in a.sizes.split(",")):
        best = None
        for _ in range(a.reps):
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(P)]
            runs = []
            for r in range(P):
                ev[r][0].record()
                run = fgt_points_exchange_begin(dy, dq, dx, *a.args, share=(r, P))
                ev[r][1].record()
                runs.append(run)
            _emulated_exchange(runs)
            times = []
            for r, run in enumerate(runs):
                ev[r][2].record()
                _, t = run.finish(return_times=True)
                ev[r][3].record()
                times.append(t)
            torch.cuda.synchronize()
            ms = [ev[r][0].elapsed_time(ev[r][1]) + ev[r][2].elapsed_time(ev[r][3]) for r in range(P)]
            xbytes = [sum(run.recv_counts) * run.slot * 8 for run in runs]
            if best is None or max(ms) < best[0]:
                best = (max(ms), ms, xbytes, times)
        mx, ms, xbytes, times = best
        slow = int(np.argmax(ms))
        print(json.dumps({"P": P, "mode": "exchange", "max_rank_ms": round(mx, 3),
                          "est_points_per_s": 2 * a.n / (mx * 1e-3), "rank_ms": [round(m, 3) for m in ms],
                          "halo_recv_MB": [round(b / 1e6, 1) for b in xbytes],
                          "slowest": {k: round(times[slow][k], 3) for k in ("tree_ms", "lists_ms", "form_ms",
                                                                            "gather_ms", "eval_ms", "direct_ms")}}))


def sequential_probe(a, dy, dq, dx):
    """Exchange path, one rank at a time (begin -> zero halo of the exchanged size -> finish),
    CUDA-event time per rank; a full run per rank is freed before the next one starts."""
    from paper_2305_07165_b200.point_fgt import fgt_points_exchange_begin
    res = []
    for P in (int(s) for s in a.sizes.split(",")):
        ms, xbytes, times = [], [], []
        for r in range(P):
            best = None
            for _ in range(a.reps):
                e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                e[0].record()
                run = fgt_points_exchange_begin(dy, dq, dx, *a.args, share=(r, P))
                e[1].record()
                recv = torch.zeros(sum(run.recv_counts) * run.slot, dtype=torch.float64, device="cuda")
                run.unpack(recv)
                e[2].record()
                _, t = run.finish(return_times=True)
                e[3].record()
                torch.cuda.synchronize()
                m = e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3])
                if best is None or m < best[0]:
                    best = (m, sum(run.recv_counts) * run.slot * 8, t)
                del run, recv
                torch.cuda.empty_cache()
            ms.append(best[0])
            xbytes.append(best[1])
            times.append(best[2])
        slow = int(np.argmax(ms))
        line = {"P": P, "mode": "sequential (exchange path, zero halo)", "config": a.config,
                "max_rank_ms": round(max(ms), 3), "est_points_per_s": 2 * a.n / (max(ms) * 1e-3),
                "rank_ms": [round(m, 3) for m in ms], "halo_recv_MB": [round(b / 1e6, 1) for b in xbytes],
                "slowest": {k: round(times[slow][k], 3) for k in ("tree_ms", "lists_ms", "form_ms", "gather_ms",
                                                                  "eval_ms", "direct_ms")}}
        print(json.dumps(line), flush=True)
        res.append(line)
    return res


if __name__ == "__main__":
    main()
