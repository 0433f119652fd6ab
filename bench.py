#!/usr/bin/env python
"""Benchmark of the discrete plane-wave FGT hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (N=1): BASELINE.json configs[1] ("config 2"): d=3 free space, N=M=10^6,
sources from 8 isotropic Gaussian clusters (sigma 0.02, clipped to the unit box),
uniform targets, standard-normal charges, delta=1e-4, eps=1e-9, s=200.  Inputs are
generated with the SURVEY.md §8(d) recipe (numpy default_rng seeds 1 and 2).

A step is one full transform: tree + lists + form + gather + eval + direct.
`value`   = (N+M) points/s with inputs resident in HBM (fgt_points_device), CUDA events
            on the launching stream, L2 flushed (512 MB write) between steps.
`e2e`     = same metric through the host API fgt_points(): pinned host inputs copied
            H2D and potentials copied D2H inside every timed step.
`roofline`= the dominant kernel (the FP64-tensor-core form kernel): algorithmic
            flops 8*N_F per source in a P-box / its CUDA-event time, against the
            measured FP64 DMMA peak of this GPU.
Under torchrun (N>1) each rank evaluates a cost-balanced contiguous share of the
target leaves of the same problem (strong scaling; tree replicated, P-box halo
recomputed, no data-path collective); time = max over ranks.
`--impl reference` times the CPU oracle (numpy restatement of the reference; the
reference ships no compiled path) on a bounded, extrapolated sample of the same
workload, on rank 0 only.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FGT (N+M) points/sec at fixed ε on 1/2/4/8 B200; % of HBM/FP64 roofline"
CFG = dict(N=1_000_000, M=1_000_000, d=3, delta=1e-4, eps=1e-9, n_s=200, boundary="free")
WORKLOAD = ("config2: discrete free-space FGT, d=3, N=M=1e6, sources 8 Gaussian clusters "
            "(sigma=0.02, clipped), uniform targets, delta=1e-4, eps=1e-9, s=200")


def gen_config2(N, M):
    """SURVEY.md §8(d) item 2 generator."""
    r = np.random.default_rng(1)
    C = r.uniform(-0.5, 0.5, (8, 3))
    lab = r.integers(0, 8, N)
    y = np.clip(C[lab] + 0.02 * r.standard_normal((N, 3)), -0.5, 0.5)
    q = r.standard_normal(N)
    x = np.random.default_rng(2).uniform(-0.5, 0.5, (M, 3))
    return y, q, x


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()
                self.out, _ = self.p.communicate()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ CPU oracle sample
def oracle_sample(y, q, x, seed, budget=(2.0, 2.0, 1.0)):
    """Time the CPU oracle (restated reference Alg 2) on config 2: the full tree, then
    random samples of P-boxes (form), psi boxes (gather+eval) and direct target
    leaves, each extrapolated by its work share.  Returns (seconds, description)."""
    from oracle import point_fgt as op
    rng = np.random.default_rng(seed)
    a = op.Alg2(y, q, x, CFG["delta"], CFG["eps"], CFG["n_s"], CFG["boundary"])
    t0 = time.perf_counter()
    t = a.build_tree()
    t_tree = time.perf_counter() - t0

    def sample(items, weight, fn, limit):
        order = rng.permutation(len(items))
        done_w, t_spent = 0.0, 0.0
        for i in order:
            s = time.perf_counter()
            fn(items[i])
            t_spent += time.perf_counter() - s
            done_w += weight[i]
            if t_spent >= limit:
                break
        total = float(np.sum(weight))
        return t_spent * (total / done_w if done_w else 0.0), done_w / total if total else 1.0

    dense = a.dense
    w_form = t.src_count[dense].astype(float) + 1.0
    t_form, f_form = sample(dense, w_form, lambda S: a.form([S]), budget[0])
    # gather+eval cost does not depend on the expansion values: use zeros for P-boxes
    # whose expansions were not sampled
    zero = np.zeros((a.pw.n_f,) * a.dim, dtype=np.complex128)
    for S in dense:
        a.phi.setdefault(S, zero)
    psi_boxes = np.array([T for T in a.tleaves if t.level[T] == t.l_c and
                          any(a.is_dense[S] for S, _ in a.list_of(T))])
    w_ge = np.array([t.tgt_count[T] + 1.0 for T in psi_boxes])
    t_ge, f_ge = sample(psi_boxes, w_ge, lambda T: a.gather_eval([T]), budget[1])
    w_d = np.array([t.tgt_count[T] * sum(t.src_count[S] for S, _ in a.list_of(T)
                                         if not a.is_dense[S]) + 1.0 for T in a.tleaves])
    t_dir, f_dir = sample(a.tleaves, w_d, lambda T: a.direct([T]), budget[2])
    total = t_tree + t_form + t_ge + t_dir
    desc = (f"config-2 input, full oracle tree ({t_tree:.1f} s) + random samples "
            f"extrapolated by work share: form {100 * f_form:.2f}% of P-box sources, "
            f"gather+eval {100 * f_ge:.1f}% of psi boxes, direct {100 * f_dir:.1f}% of pairs; "
            f"extrapolated total {total:.0f} s")
    return total, desc


# ------------------------------------------------------------------ roofline accounting
HBM_PEAK_GBS = 6555.5  # MEASURED_PEAKS.json hbm_gbs (copy test)


def box_dft_cmacs(d, G, n_f):
    """Complex MACs of the separable grid<->mode transform of one box (real x complex
    counted as half) onto the stored half spectrum (d >= 2: h = n_f/2 + 1 axis-0 planes,
    axis 0 contracted first; k_nufft.cu)."""
    g, n, h = float(G), float(n_f), float(n_f // 2 + 1)
    if d == 1:
        return n * g
    if d == 2:
        return 0.5 * g * g * n + h * n * g
    return 0.5 * g ** 3 * h + h * g * g * n + h * n * g * n


def stored_modes(d, n_f):
    """Modes stored per expansion: the Hermitian half spectrum for d >= 2 (k_pw.cuh)."""
    return n_f ** d if d == 1 else (n_f // 2 + 1) * n_f ** (d - 1)


def kernel_rooflines(phases, fp64_peak_tf, d=3):
    """Algorithmic flops/bytes of the hot kernels over their CUDA-event
    time, averaged over the timed steps.  Exact tensor-factored sums: 8 N_F flops per
    point (one complex MAC per mode).  NUFFT path: per point 2 W^d (spread/interp FMA)
    + d W c_exp (c_exp = 20 flops per kernel exp), per box 8 x the separable-DFT complex
    MACs.  Gather: 16 B per mode per P-box read + per psi box written (compulsory).  N_F
    counts the stored (half-spectrum) modes: the work the algorithm needs for real
    charges, not the full n_f^d grid."""
    ph = phases[-1]
    w, G = ph["nufft_w"], ph["nufft_G"]
    n_f = round(ph["n_modes"] ** (1.0 / d))
    NF = stored_modes(d, n_f)
    exact_src = ph["n_src_dense"] - ph["n_src_spread"]
    exact_tgt = ph["n_tgt_psi"] - ph["n_tgt_spread"]
    per_pt = 2.0 * w ** d + d * w * 20.0
    dft = 8.0 * box_dft_cmacs(d, G, n_f)
    f_form = 8.0 * NF * exact_src + per_pt * ph["n_src_spread"] + dft * ph["n_spread_boxes"]
    f_eval = 8.0 * NF * exact_tgt + per_pt * ph["n_tgt_spread"] + dft * ph["n_spread_psi"]
    # compulsory bytes: every phi read once, every psi written once; the
    # per-P-entry streamed count (16 N_F per entry) exceeds what the sibling-group kernel
    # actually moves, so it is not used as the roofline numerator
    b_gather = 16.0 * NF * (ph["n_dense"] + ph["n_psi"])
    mean = lambda k: float(np.mean([p[k] for p in phases]))  # noqa: E731
    src = "FP64 DMMA microbenchmark on this GPU (fgt_bench_fp64_peak; not in MEASURED_PEAKS.json)"
    out = []
    for name, alg, ms, bound in (
            ("form (exact DMMA sums + ES-kernel NUFFT)", f_form, mean("k_form_ms"), "tensor"),
            ("eval (exact DMMA sums + ES-kernel NUFFT)", f_eval, mean("k_eval_ms"), "tensor"),
            ("gather_kernel (diagonal translation)", b_gather, mean("k_gather_ms"), "hbm")):
        if ms <= 0:
            continue
        if bound == "tensor":
            ach = alg / (ms * 1e-3) / 1e12
            out.append({"kernel": name, "bound": "tensor", "achieved": ach, "peak": fp64_peak_tf,
                        "unit": "TFLOP/s", "frac": ach / fp64_peak_tf, "kernel_ms": ms, "alg": alg,
                        "accounting": "algorithmic FP64 flops per launch", "peak_source": src})
        else:
            ach = alg / (ms * 1e-3) / 1e9
            out.append({"kernel": name, "bound": "hbm", "achieved": ach, "peak": HBM_PEAK_GBS,
                        "unit": "GB/s", "frac": ach / HBM_PEAK_GBS, "kernel_ms": ms, "alg": alg,
                        "accounting": "compulsory bytes per launch (each phi read once, each psi written once)",
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs"})
    return out


# kernels (ncu names) that make up each CUDA-event phase of kernel_rooflines
PHASE_KERNELS = {
    "form": ("spread_pencil_kernel", "pencil_reduce_kernel", "spread_tile_kernel", "sort_records_kernel", "spread_taps_kernel", "spread_keys_kernel",
             "form_kernel", "form_reduce_kernel", "plane_reduce_kernel", "bgemm_kernel",
             "job_ranges_kernel", "DeviceRadixSort"),
    "eval": ("eval_kernel", "interp_kernel"),
    "gather": ("gather_kernel", "group_table_kernel"),
}


def phase_traffic(kernel_label):
    """DRAM bytes (read + write) per step of the kernels of a phase, from the newest
    committed `ncu --set full` summary of the same workload (profiles/r*_ncu_kernels.json,
    tools/ncu_summary.py); None if there is none."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_kernels.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        rep = json.load(f)
    if not isinstance(rep, dict) or "kernels" not in rep:
        return None
    phase = kernel_label.split(" ")[0].split("_")[0]
    pats = PHASE_KERNELS.get(phase)
    if not pats:
        return None
    tot = 0.0
    for k in rep["kernels"]:
        if any(p in k["kernel"] for p in pats):
            tot += k.get("dram__bytes_read.sum [GB]", 0.0) + k.get("dram__bytes_write.sum [GB]", 0.0)
    return {"bytes": tot * 1e9 / rep.get("steps", 1), "source": os.path.basename(files[-1]),
            "kernels": list(pats)}


# ------------------------------------------------------------------ distributed helpers
def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ arms
def run_reference(args, world, rank):
    if rank != 0:
        return None
    y, q, x = gen_config2(CFG["N"], CFG["M"])
    times, desc = [], ""
    for s in range(args.warmup + args.steps):
        tot, desc = oracle_sample(y, q, x, seed=s)
        if s >= args.warmup:
            times.append(tot)
    sec = float(np.mean(times))
    value = (CFG["N"] + CFG["M"]) / sec
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (config-2 generator, seeds 1/2)",
        "config": {"workload": WORKLOAD, **CFG},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": 1, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def run_ours(args, world, rank, local):
    import torch
    from paper_2305_07165_b200 import _lib, fgt_points, fgt_points_device
    from paper_2305_07165_b200.point_fgt import FgtParams
    import ctypes

    lib = _lib.load()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    N, M = args.n or CFG["N"], args.n or CFG["M"]
    y, q, x = gen_config2(N, M)
    share = (rank, world)
    prm = FgtParams(3, CFG["delta"], CFG["eps"], CFG["n_s"], False, share)
    dy, dq, dx = (torch.from_numpy(a).to(dev) for a in (y, q, x))
    u = torch.empty(M, dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    from paper_2305_07165_b200.point_fgt import PointsRun, TorchExchange
    xchg = TorchExchange()

    def step(sy=dy, sq=dq, sx=dx, out=u):
        if world == 1:
            return fgt_points_device(sy, sq, sx, CFG["delta"], CFG["eps"], CFG["n_s"], out=out,
                                     params=prm, return_times=True)[1]
        # multi-GPU: each rank forms the expansions it owns; the one-box halo of
        # expansions goes over NCCL (one all-to-all), then translation/evaluation/near field
        run = PointsRun(prm, sy, sq, sx)
        run.exchange(xchg)
        return run.finish(out=out, return_times=True)[1]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-resident timed region
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    phases = []
    barrier(world)
    torch.cuda.synchronize()
    l0 = lib.fgt_launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))          # L2 flush, outside the events
            ev[i][0].record(stream)
            phases.append(step())
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = lib.fgt_launch_count() - l0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = max_over_ranks(float(np.sum(step_ms)), world)
    ms_per_step = total_ms / args.steps
    value = (N + M) / (ms_per_step * 1e-3)

    # ---- end-to-end through the host API (pinned host buffers, H2D + D2H per step)
    hy, hq, hx = (torch.from_numpy(a).pin_memory() for a in (y, q, x))
    hu = torch.empty(M, dtype=torch.float64).pin_memory()
    ny, nq, nx, nu = hy.numpy(), hq.numpy(), hx.numpy(), hu.numpy()
    e2e_s = []

    def e2e_step():
        if world == 1:
            return fgt_points(ny, nq, nx, CFG["delta"], CFG["eps"], CFG["n_s"], share=share, out=nu)
        ey, eq, ex = (t.to(dev, non_blocking=True) for t in (hy, hq, hx))
        step(ey, eq, ex, u)
        hu.copy_(u, non_blocking=True)
        torch.cuda.synchronize()
        return nu

    for _ in range(args.warmup):  # the host path owns its own stream: warm it up too
        e2e_step()
    barrier(world)
    for i in range(max(1, args.steps)):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res_u = e2e_step()
        e2e_s.append(time.perf_counter() - t0)
    if res_u is not nu:
        nu[:] = res_u
    barrier(world)
    e2e_sec = max_over_ranks(float(np.mean(e2e_s)), world)
    h2d = (y.nbytes + q.nbytes + x.nbytes)
    d2h = M * 8

    # ---- rooflines of the hot kernels; the dominant one (by device time) is reported
    ph = phases[-1]
    peak = ctypes.c_double()
    _lib.check(lib.fgt_bench_fp64_peak(1, ctypes.byref(peak)))
    kr = kernel_rooflines(phases, peak.value)
    dom = max(kr, key=lambda k: k["kernel_ms"])
    traffic = phase_traffic(dom["kernel"])

    res = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (config-2 generator, seeds 1/2)",
        "config": {"workload": WORKLOAD, **CFG, "N": N, "M": M,
                   "parallelism": (f"target-leaf shares x{world}, owner-formed expansions, one-box halo "
                                   "over NCCL all-to-all" if world > 1 else "single GPU"),
                   "l2": "flushed between steps (512 MB write, untimed)"},
        "e2e": {"value": (N + M) / e2e_sec, "unit": "points/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_sec * 1e3},
        "roofline": {**{k: dom[k] for k in ("bound", "achieved", "peak", "unit", "frac")},
                     "traffic": traffic["bytes"] if traffic else None,
                     "traffic_unit": "bytes per step (dram read + write, ncu --set full)",
                     "traffic_source": traffic, "kernel": dom["kernel"], "kernel_ms": dom["kernel_ms"],
                     "alg_per_launch": dom["alg"], "accounting": dom["accounting"],
                     "peak_source": dom["peak_source"]},
        "kernels": kr,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "phases_ms": {k: ph[k] for k in ("tree_ms", "lists_ms", "form_ms", "gather_ms",
                                          "eval_ms", "direct_ms", "k_form_ms", "k_gather_ms",
                                          "k_eval_ms", "k_direct_ms")},
        "work": {k: ph[k] for k in ("n_boxes", "n_dense", "n_psi", "n_src_dense", "n_tgt_psi",
                                     "n_p_entries", "n_direct_pairs", "n_modes", "n_spread_boxes",
                                     "n_src_spread", "n_spread_psi", "n_tgt_spread", "nufft_w",
                                     "nufft_G")},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sec, desc = oracle_sample(y, q, x, seed=0)
        res["cpu_baseline"] = {"value": (N + M) / sec, "unit": "points/s", "cores": 1,
                               "kind": "port", "sample": desc}
    if rank == 0 and world == 1 and not args.no_volume:
        res["volume"] = run_volume_leg(args, flush)
    return res


def run_volume_leg(args, flush):
    """Secondary line: BASELINE configs[3] (volume FGT, d=3, k=16, delta=1e-4, eps=1e-10,
    5 Gaussians): device time of fgt_box_device per step (plan prebuilt), grid points/s;
    e2e adds the host plan and the H2D/D2H of the leaf grids."""
    import torch
    from paper_2305_07165_b200 import volume as pv
    from tools.prof_volume import build
    tree, vals, plan, t_tree, t_plan = build()
    from tools.prof_volume import config4_density_torch
    t0 = time.perf_counter()
    tree_g, _, _ = pv.build_density_tree(config4_density_torch(), 3, 16, 1e-10, device="cuda")
    t_tree_gpu = time.perf_counter() - t0
    same_tree = bool(np.array_equal(tree_g.level, tree.level) and np.array_equal(tree_g.coords, tree.coords))
    leaves, V = pv._stack_values(tree, vals, 16)
    dv = torch.from_numpy(V).cuda()
    out = torch.empty_like(dv)
    for _ in range(3):
        pv.fgt_box_device(plan, dv, out)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ms, ph = [], None
    for i in range(args.steps):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        _, ph = pv.fgt_box_device(plan, dv, out, return_times=True)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    npts = V.size
    t0 = time.perf_counter()
    u = pv.fgt_box(tree, vals, 1e-4, 1e-10)
    e2e = time.perf_counter() - t0
    # same with the plan reused (repeated transforms on one tree): H2D + GPU + D2H
    pv.fgt_box(tree, vals, 1e-4, 1e-10, plan=plan)
    t0 = time.perf_counter()
    pv.fgt_box(tree, vals, 1e-4, 1e-10, plan=plan)
    e2e_reuse = time.perf_counter() - t0
    cpu = None
    if not args.no_cpu_baseline:
        # oracle Alg 4 on a coarser tree of the same density and parameters (tree eps 1e-4:
        # ~340 leaves, same k and n_f, so the per-grid-point cost is representative)
        from oracle import volume as ov
        from tools.prof_volume import config4_density
        otree = ov.density_tree(config4_density(), 3, 16, 1e-4)
        t0 = time.perf_counter()
        ov.fgt_box(otree, 1e-4, 1e-10)
        sec = time.perf_counter() - t0
        on = int(otree.is_leaf.sum()) * 16 ** 3
        cpu = {"value": on / sec, "unit": "grid points/s", "cores": 1, "kind": "port",
               "sample": f"oracle Alg 4 (numpy) on the config-4 density with tree eps 1e-4: "
                         f"{int(otree.is_leaf.sum())} leaves = {on} grid points, {sec:.1f} s"}
    return {"workload": "config4: volume FGT d=3, k=16, 5 Gaussians (w 0.01-0.1), "
                        "delta=1e-4, eps=1e-10, tree eps 1e-10",
            "metric": "grid points/s (N = N_leaf k^d)", "grid_points": int(npts),
            "n_leaves": int(len(leaves)), "n_boxes": int(tree.n_boxes),
            "value": npts / (float(np.mean(ms)) * 1e-3), "ms_per_step": float(np.mean(ms)),
            "e2e": {"value": npts / e2e, "ms_per_step": e2e * 1e3,
                    "includes": "host tables/schedules + H2D + GPU + D2H"},
            "e2e_plan_reused": {"value": npts / e2e_reuse, "ms_per_step": e2e_reuse * 1e3,
                                "includes": "H2D + GPU + D2H (BoxPlan built once per tree)"},
            "cpu_baseline": cpu,
            "host_density_tree_s": t_tree, "host_plan_s": t_plan,
            "density_tree_gpu_sigma_s": t_tree_gpu, "density_tree_gpu_sigma_same_tree": same_tree,
            "phases_ms": {k: ph[k] for k in ("form_ms", "gather_ms", "eval_ms", "direct_ms")},
            "checksum": float(sum(np.sum(v) for v in u.values()))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=0, help="override N=M (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-volume", action="store_true", help="skip the config-4 volume leg")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        res = run_reference(args, world, rank)
    else:
        res = run_ours(args, world, rank, local)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
