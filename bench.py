#!/usr/bin/env python
"""Benchmark of the discrete plane-wave FGT hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 5]

Headline workload (N=1): BASELINE.json configs[4] ("config 5", the configuration BASELINE
quotes at 1/2/4/8 GPUs; it fits one B200): d=3 free space, N=M=10^8, sources on a
spherical shell (r=0.35, thickness 1e-3), uniform targets, charges U[-1,1],
delta=1e-6, eps=1e-6, s=256.  Inputs follow the SURVEY.md §8(d) recipe (numpy
default_rng seeds 0 and 1; tools/configs.py).  Configs 2 and 3 (and the volume config 4)
are reported as secondary lines under "extra".

A step is one full transform: tree + lists + form + gather + eval + direct.
`value`    (N+M) points/s with inputs resident in HBM (fgt_points_device), CUDA events on
           the launching stream; inputs (6.4 GB) exceed L2, and L2 is also flushed
           (512 MB write, untimed) between steps.
`e2e`      same metric through the host API fgt_points(): pinned host inputs copied H2D
           and potentials copied D2H inside every timed step.
`check`    after the timed steps, u at 1000 random targets vs a CPU fp64 Gaussian sum over
           every source within r^2 = 40 delta (oracle/nearsum.py); the run fails above
           10 eps.
`roofline` the dominant phase by device time (the form at config 5): algorithmic FP64
           flops over its CUDA-event time vs the FP64 DMMA peak this
           library measures on the GPU (MEASURED_PEAKS.json has no FP64 entry); HBM
           phases use MEASURED_PEAKS.json hbm_gbs.
`cpu_baseline`  the CPU oracle (numpy restatement of the reference Alg 2) run on
           bounded samples of the same workload, one sample per host core in parallel
           processes (see `shell_samples`), measured wall time.
Under torchrun (N>1) every rank runs the same problem and evaluates a cost-balanced
contiguous Morton range of the target leaves; each rank forms only the P-box expansions
it owns, the one-box halo of expansions is exchanged with one NCCL all-to-all and the
potentials are assembled on every rank with one NCCL all-reduce (PointsRun +
TorchExchange); time = max over ranks ("scaling": "strong").
`--impl reference` times the CPU oracle alone (rank 0; other ranks exit 0) on the same
samples: every step is one parallel round of full oracle transforms, measured.
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

from tools import configs  # noqa: E402

METRIC = "FGT (N+M) points/sec at fixed ε on 1/2/4/8 B200; % of HBM/FP64 roofline"


# ------------------------------------------------------------------ host / peaks
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def hbm_peak():
    """MEASURED_PEAKS.json hbm_gbs (driver-written); the profiling recipe's fallback if absent."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


FP64_SRC = ("FP64 DMMA (mma.sync m8n8k4 f64) microbenchmark run by this bench on this GPU "
            "(fgt_bench_fp64_peak); MEASURED_PEAKS.json has no FP64 entry")


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
                 "--format=csv,noheader,nounits", "-lms", "250"],
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


# ------------------------------------------------------------------ CPU oracle samples
_SAMPLES = []


def shell_samples(y, q, x, n, seed=7, L_s=0.016):
    """n disjoint bounded samples of config 5, each a self-contained problem whose
    per-point work mix matches the full transform: the sources and targets inside a cube
    of side L_s centred on a random shell point (a ~20k-source shell patch: P-boxes
    with ~800 sources, their colleagues, ~6-target psi boxes, near field), plus the
    targets of a source-free cube inside the sphere sized so the sample holds as many
    targets as sources (config 5 has N = M).  The cutoff box side is D0 sqrt(delta)
    whatever the sample's extent, so every box does the work it does in the full run;
    only the boxes on the cube faces lose their outside neighbours."""
    r = np.random.default_rng(seed)
    out = []

    def inside(p, c, L):
        m = np.abs(p[:, 0] - c[0]) < L / 2
        i = np.nonzero(m)[0]
        return i[np.all(np.abs(p[i] - c) < L / 2, axis=1)]

    for _ in range(n):
        d = r.standard_normal(3)
        c = 0.35 * d / np.linalg.norm(d)
        i = inside(y, c, L_s)
        j = inside(x, c, L_s)
        need = max(0, i.size - j.size)
        L_t = (need / x.shape[0]) ** (1.0 / 3.0)
        ct = r.uniform(-0.15, 0.15, 3)
        jt = inside(x, ct, L_t) if need else np.zeros(0, np.int64)
        out.append((y[i].copy(), q[i].copy(), np.vstack([x[j], x[jt]])))
    return out


def _oracle_worker(k):
    from threadpoolctl import threadpool_limits
    from oracle import point_fgt as op
    cfg = configs.CONFIGS[5]
    ys, qs, xs = _SAMPLES[k]
    with threadpool_limits(1):
        t0 = time.perf_counter()
        op.fgt_points(ys, qs, xs, cfg["delta"], cfg["eps"], cfg["n_s"], cfg["boundary"])
        return time.perf_counter() - t0


class OracleRunner:
    """One process per host core (fork), each owning one sample; a step runs every
    sample once in parallel and is timed by the wall clock around the whole round."""

    def __init__(self, y, q, x, procs=None):
        import multiprocessing as mp
        self.procs = procs or os.cpu_count() or 1
        global _SAMPLES
        _SAMPLES = shell_samples(y, q, x, self.procs)
        self.points = int(sum(a.shape[0] + c.shape[0] for a, _, c in _SAMPLES))
        self.sources = int(sum(a.shape[0] for a, _, _ in _SAMPLES))
        self.pool = mp.get_context("fork").Pool(self.procs)

    def step(self):
        t0 = time.perf_counter()
        per = self.pool.map(_oracle_worker, range(self.procs), chunksize=1)
        return time.perf_counter() - t0, per

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self, sec):
        return (f"{self.procs} parallel processes (one per host core, BLAS 1 thread each), each a "
                f"full oracle Alg 2 transform of one config-5 sample (shell patch in a 0.016 cube + "
                f"as many far targets as sources): {self.points} points ({self.sources} sources) "
                f"per step, {sec:.2f} s wall; host {cpu_model()}, nproc {os.cpu_count()}")


# ------------------------------------------------------------------ roofline accounting
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


def kernel_rooflines(phases, fp64_peak_tf, hbm_gbs, d):
    """Algorithmic flops/bytes of the hot phases over their CUDA-event
    time, averaged over the timed steps.  Exact tensor-factored sums: 8 N_F flops per
    point (one complex MAC per stored mode).  NUFFT path: per point 2 W^d (spread/interp
    FMA) + d W c_exp (c_exp = 20 flops per kernel exp), per box 8 x the separable-DFT
    complex MACs.  Gather: 16 B per stored mode per P-box read + per psi box written
    (compulsory).  Direct: 3d+3+20 flops per pair (c_exp = 20)."""
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
    b_gather = 16.0 * NF * (ph["n_dense"] + ph["n_psi"])
    f_direct = (3.0 * d + 3.0 + 20.0) * ph["n_direct_pairs"]
    mean = lambda k: float(np.mean([p[k] for p in phases]))  # noqa: E731
    out = []
    # fused translation + evaluation (psi never stored): the gather phase holds only the group
    # table (its time could not move the compulsory phi + psi bytes at the HBM peak), so the
    # translation's 8 N_F flops per P-list entry count with the
    # evaluation kernel that performs them and there is no separate gather line
    fused = mean("k_gather_ms") > 0 and b_gather / (mean("k_gather_ms") * 1e-3) / 1e9 > hbm_gbs
    eval_name = "eval (exact DMMA sums + ES-kernel NUFFT)"
    if fused:
        f_eval += 8.0 * NF * ph["n_p_entries"]
        b_gather = 0.0
        eval_name = "translation + eval (fused: psi never stored; exact DMMA sums)"
    for name, alg, ms, bound in (
            ("form (exact DMMA sums + ES-kernel NUFFT: taps, records, pencils, DFT stages)", f_form,
             mean("k_form_ms"), "tensor"),
            (eval_name, f_eval, mean("k_eval_ms"), "tensor"),
            ("gather (diagonal translation)", b_gather, mean("k_gather_ms"), "hbm"),
            ("direct (near field, ball cut)", f_direct, mean("k_direct_ms"), "fp64")):
        if ms <= 0 or alg <= 0:
            continue
        if bound in ("tensor", "fp64"):
            ach = alg / (ms * 1e-3) / 1e12
            out.append({"kernel": name, "bound": "tensor" if bound == "tensor" else "fp64",
                        "achieved": ach, "peak": fp64_peak_tf, "unit": "TFLOP/s",
                        "frac": ach / fp64_peak_tf, "kernel_ms": ms, "alg": alg,
                        "accounting": "algorithmic FP64 flops per launch", "peak_source": FP64_SRC})
        else:
            ach = alg / (ms * 1e-3) / 1e9
            out.append({"kernel": name, "bound": "hbm", "achieved": ach, "peak": hbm_gbs,
                        "unit": "GB/s", "frac": ach / hbm_gbs, "kernel_ms": ms, "alg": alg,
                        "accounting": "compulsory bytes per launch (each phi read once, each psi written once)",
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs"})
    return out


# kernels (ncu names) that make up each CUDA-event phase of kernel_rooflines
PHASE_KERNELS = {
    "form": ("spread_pencil_kernel", "pencil_reduce_kernel", "pencil_jobs_kernel", "gather_jobs_kernel",
             "spread_tile_kernel", "sort_records_kernel", "spread_taps_kernel", "spread_keys_kernel",
             "form_kernel", "form_reduce_kernel", "plane_reduce_kernel", "bgemm_kernel", "dft3_fused_kernel",
             "job_ranges_kernel"),
    "eval": ("eval_kernel", "interp_kernel", "gather_eval_kernel"),
    "translation": ("eval_kernel", "interp_kernel", "gather_eval_kernel"),
    "direct": ("direct_warp_kernel", "direct_kernel"),
    "gather": ("gather_kernel", "group_table_kernel"),
}


def phase_traffic(kernel_label, cfg_id):
    """DRAM bytes (read + write) per step of the kernels of a phase, from the newest
    committed `ncu --set full` summary of the same workload
    (profiles/r*_c{cfg}_ncu_kernels.json, tools/ncu_summary.py); None if there is none."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_c{cfg_id}_ncu_kernels.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        rep = json.load(f)
    if not isinstance(rep, dict) or "kernels" not in rep:
        return None
    pats = PHASE_KERNELS.get(kernel_label.split(" ")[0])
    if not pats:
        return None
    tot = 0.0
    for k in rep["kernels"]:
        if any(p in k["kernel"] for p in pats):
            tot += k.get("dram__bytes_read.sum [GB]", 0.0) + k.get("dram__bytes_write.sum [GB]", 0.0)
    return {"bytes": tot * 1e9 / rep.get("steps", 1), "source": os.path.basename(files[-1]),
            "kernels": list(pats)}


# ------------------------------------------------------------------ distributed helpers
def dist_setup():
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


def config_block(cfg_id, N, M, world):
    cfg = configs.CONFIGS[cfg_id]
    return {"workload": configs.WORKLOADS[cfg_id], "config_id": cfg_id, "d": cfg["d"], "N": N, "M": M,
            "delta": cfg["delta"], "eps": cfg["eps"], "n_s": cfg["n_s"], "boundary": cfg["boundary"],
            "parallelism": (f"target-leaf shares x{world}, owner-formed expansions, one-box halo over "
                            "NCCL all-to-all" if world > 1 else "single GPU"),
            "l2": "inputs larger than L2; also flushed between steps (512 MB write, untimed)"}


# ------------------------------------------------------------------ arms
def run_reference(args):
    """CPU oracle arm: rank 0 only (the other ranks exit 0 without work)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return None
    y, q, x = configs.generate(5)
    runner = OracleRunner(y, q, x)
    del y, q, x
    times = []
    for s in range(args.warmup + args.steps):
        sec, _ = runner.step()
        if s >= args.warmup:
            times.append(sec)
    runner.close()
    sec = float(np.mean(times))
    value = runner.points / sec
    desc = runner.describe(sec)
    cfg = configs.CONFIGS[5]
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (config-5 generator, seeds 0/1)",
        "config": config_block(5, cfg["N"], cfg["M"], 1),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": runner.procs, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host": {"cpu": cpu_model(), "nproc": os.cpu_count()},
    }


def check_result(u_host, y, q, x, cfg, n=1000, seed=99):
    """u at n random targets vs the CPU fp64 ball-restricted exact sum (oracle/nearsum.py)."""
    from oracle.nearsum import near_sum
    sub = np.sort(np.random.default_rng(seed).choice(x.shape[0], min(n, x.shape[0]), replace=False))
    t0 = time.perf_counter()
    ex = near_sum(y, q, x[sub], cfg["delta"], cfg["boundary"] == "periodic")
    err = float(np.linalg.norm(u_host[sub] - ex) / max(np.linalg.norm(ex), 1e-300))
    return {"targets": int(sub.size), "rel_l2": err, "bar_10eps": 10 * cfg["eps"],
            "pass": bool(err <= 10 * cfg["eps"]), "reference": "CPU fp64 sum over all sources within "
            "r^2 = 40 delta (oracle/nearsum.py)", "check_s": time.perf_counter() - t0}


def timed_device_steps(step, steps, flush, stream, lib, local, world):
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    phases = []
    barrier(world)
    torch.cuda.synchronize()
    l0 = lib.fgt_launch_count()
    with ClockSampler(local) as clk:
        # more untimed steps for ~1 s while nvidia-smi starts (its NVML initialisation stalls
        # kernel launches for tens of ms once: it showed as a single 270-285 ms step among
        # 243 ms ones when the sampler started with the first timed step)
        t_start = time.perf_counter()
        while True:
            step()
            torch.cuda.synchronize()
            # (every rank must run the same number of steps: the decision is all-reduced)
            if max_over_ranks(1.0 if time.perf_counter() - t_start > 1.0 else 0.0, world) > 0.5:
                break
        barrier(world)
        torch.cuda.synchronize()
        l0 = lib.fgt_launch_count()
        for i in range(steps):
            flush.fill_(float(i))          # L2 flush, outside the events
            ev[i][0].record(stream)
            phases.append(step())
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = lib.fgt_launch_count() - l0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    return step_ms, phases, launches, clk.summary()


def run_ours(args, world, rank, local):
    import ctypes
    import torch
    from paper_2305_07165_b200 import _lib, fgt_points, fgt_points_device
    from paper_2305_07165_b200.point_fgt import FgtParams, PointsRun, TorchExchange

    lib = _lib.load()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cid = args.config
    cfg = configs.CONFIGS[cid]
    N = args.n or cfg["N"]
    M = args.n or cfg["M"]
    t_gen = time.perf_counter()
    y, q, x = configs.generate(cid, N, M)
    t_gen = time.perf_counter() - t_gen
    share = (rank, world)
    prm = FgtParams(cfg["d"], cfg["delta"], cfg["eps"], cfg["n_s"], cfg["boundary"] == "periodic", share)
    dy, dq, dx = (torch.from_numpy(a).to(dev) for a in (y, q, x))
    u = torch.empty(M, dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    xchg = TorchExchange()
    args3 = (cfg["delta"], cfg["eps"], cfg["n_s"], cfg["boundary"])

    def step(sy=dy, sq=dq, sx=dx, out=u):
        if world == 1:
            return fgt_points_device(sy, sq, sx, *args3, out=out, params=prm, return_times=True)[1]
        # multi-GPU: each rank forms the expansions it owns; the one-box halo of
        # expansions goes over NCCL (one all-to-all), then translation/evaluation/near field
        run = PointsRun(prm, sy, sq, sx)
        run.exchange(xchg)
        ph = run.finish(out=out, return_times=True)[1]
        xchg.assemble(out)  # u of all targets on every rank (NCCL all-reduce of the shares)
        return ph

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-resident timed region
    step_ms, phases, launches, clocks = timed_device_steps(step, args.steps, flush, stream, lib,
                                                           local, world)
    total_ms = max_over_ranks(float(np.sum(step_ms)), world)
    ms_per_step = total_ms / args.steps
    value = (N + M) / (ms_per_step * 1e-3)

    # ---- result check (outside the timed region): this rank's share vs CPU exact sums
    u_host = u.cpu().numpy()   # multi-GPU: already assembled on every rank by step()
    check = check_result(u_host, y, q, x, cfg) if rank == 0 else None
    if rank == 0 and not check["pass"]:
        raise SystemExit(f"bench: result check failed: {check}")

    # ---- end-to-end through the host API (pinned host buffers, H2D + D2H per step)
    hy, hq, hx = (torch.from_numpy(a).pin_memory() for a in (y, q, x))
    hu = torch.empty(M, dtype=torch.float64).pin_memory()
    ny, nq, nx, nu = hy.numpy(), hq.numpy(), hx.numpy(), hu.numpy()
    e2e_s = []

    def e2e_step():
        if world == 1:
            return fgt_points(ny, nq, nx, *args3, share=share, out=nu)
        ey, eq, ex = (t.to(dev, non_blocking=True) for t in (hy, hq, hx))
        step(ey, eq, ex, u)
        hu.copy_(u, non_blocking=True)
        torch.cuda.synchronize()
        return nu

    for _ in range(args.warmup):  # the host path owns its own stream: warm it up too
        e2e_step()
    barrier(world)
    for i in range(args.steps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        e2e_s.append(time.perf_counter() - t0)
    barrier(world)
    e2e_sec = max_over_ranks(float(np.mean(e2e_s)), world)
    e2e_err = None
    if rank == 0 and world == 1:
        e2e_err = float(np.max(np.abs(nu - u_host)))   # host path == device path (deterministic)
    h2d = y.nbytes + q.nbytes + x.nbytes
    d2h = M * 8
    del hy, hq, hx, hu, ny, nq, nx, nu

    # ---- rooflines of the hot phases; the dominant one (by device time) is reported
    peak = ctypes.c_double()
    _lib.check(lib.fgt_bench_fp64_peak(1, ctypes.byref(peak)))
    hbm, _ = hbm_peak()
    kr = kernel_rooflines(phases, peak.value, hbm, cfg["d"])
    dom = max(kr, key=lambda k: k["kernel_ms"])
    traffic = phase_traffic(dom["kernel"], cid)
    ph = phases[-1]
    res = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (config-{cid} generator, SURVEY.md §8(d) seeds)",
        "config": config_block(cid, N, M, world),
        "e2e": {"value": (N + M) / e2e_sec, "unit": "points/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_sec * 1e3,
                "max_abs_diff_vs_device_path": e2e_err},
        "check": check,
        "roofline": {**{k: dom[k] for k in ("bound", "achieved", "peak", "unit", "frac")},
                     "traffic": traffic["bytes"] if traffic else None,
                     "traffic_unit": "bytes per step (dram read + write, ncu --set full)",
                     "traffic_source": traffic, "kernel": dom["kernel"], "kernel_ms": dom["kernel_ms"],
                     "alg_per_launch": dom["alg"], "accounting": dom["accounting"],
                     "peak_source": dom["peak_source"]},
        "kernels": kr,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "step_ms": {"min": float(np.min(step_ms)), "median": float(np.median(step_ms)),
                    "max": float(np.max(step_ms))},
        "phases_ms": {k: ph[k] for k in ("tree_ms", "lists_ms", "form_ms", "gather_ms",
                                          "eval_ms", "direct_ms", "k_form_ms", "k_gather_ms",
                                          "k_eval_ms", "k_direct_ms")},
        "work": {k: ph[k] for k in ("n_boxes", "n_dense", "n_psi", "n_src_dense", "n_tgt_psi",
                                     "n_p_entries", "n_direct_pairs", "n_modes", "n_spread_boxes",
                                     "n_src_spread", "n_spread_psi", "n_tgt_spread", "nufft_w",
                                     "nufft_G")},
        "host": {"cpu": cpu_model(), "nproc": os.cpu_count(), "generate_s": t_gen},
    }
    del dy, dq, dx, u
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline and cid == 5:
        runner = OracleRunner(y, q, x)
        sec, _ = runner.step()
        runner.close()
        res["cpu_baseline"] = {"value": runner.points / sec, "unit": "points/s", "cores": runner.procs,
                               "kind": "port", "sample": runner.describe(sec)}
    del y, q, x
    if rank == 0 and world == 1 and not args.no_extra:
        res["extra"] = {f"config{c}": run_extra(c, flush, args) for c in (2, 3)}
        res["extra"]["config4_volume"] = run_volume_leg(args, flush, peak.value)
    return res


def run_extra(cid, flush, args):
    """Secondary line: another point config at full size (device-resident ms/step, e2e
    through fgt_points, result check)."""
    import torch
    from paper_2305_07165_b200 import fgt_points, fgt_points_device
    cfg = configs.CONFIGS[cid]
    y, q, x = configs.generate(cid)
    dy, dq, dx = (torch.from_numpy(a).cuda() for a in (y, q, x))
    u = torch.empty(x.shape[0], dtype=torch.float64, device="cuda")
    a3 = (cfg["delta"], cfg["eps"], cfg["n_s"], cfg["boundary"])
    for _ in range(3):
        fgt_points_device(dy, dq, dx, *a3, out=u)
    torch.cuda.synchronize()
    ms = []
    for i in range(max(5, args.steps // 2)):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _, ph = fgt_points_device(dy, dq, dx, *a3, out=u, return_times=True)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    check = check_result(u.cpu().numpy(), y, q, x, cfg)
    hu = torch.empty(x.shape[0], dtype=torch.float64).pin_memory().numpy()
    hy, hq, hx = (torch.from_numpy(a).pin_memory().numpy() for a in (y, q, x))
    fgt_points(hy, hq, hx, *a3, out=hu)
    e2e = []
    for _ in range(5):
        t0 = time.perf_counter()
        fgt_points(hy, hq, hx, *a3, out=hu)
        e2e.append(time.perf_counter() - t0)
    n = y.shape[0] + x.shape[0]
    return {"workload": configs.WORKLOADS[cid], "value": n / (np.mean(ms) * 1e-3), "unit": "points/s",
            "ms_per_step": float(np.mean(ms)), "e2e": {"value": n / np.mean(e2e), "ms_per_step": 1e3 * float(np.mean(e2e))},
            "check": check, "phases_ms": {k: round(ph[k], 3) for k in ("tree_ms", "form_ms", "gather_ms", "eval_ms", "direct_ms")}}


def run_volume_leg(args, flush, fp64_peak):
    """Secondary line: BASELINE configs[3] (volume FGT, d=3, k=16, delta=1e-4, eps=1e-10,
    5 Gaussians): device time of fgt_box_device per step (plan prebuilt), grid points/s;
    roofline = algorithmic FP64 flops of the per-axis contractions (SURVEY.md §8(d) K5:
    2 n_f k^3 + 8 (n_f^2 k^2 + n_f^3 k) per leaf->PW and per PW->grid, 2 d k^(d+1) per
    direct pair) over the whole transform's device time."""
    import torch
    from paper_2305_07165_b200 import volume as pv
    from tools.prof_volume import build, config4_density_torch
    tree, vals, plan, t_tree, t_plan = build()
    t0 = time.perf_counter()
    tree_g, _, _ = pv.build_density_tree(config4_density_torch(), 3, 16, 1e-10, device="cuda")
    t_tree_gpu = time.perf_counter() - t0
    # same box set (the device build numbers the boxes its balance sweeps create in sweep order)
    canon = lambda t: sorted(map(tuple, np.column_stack([t.level, t.coords, t.is_leaf]).tolist()))  # noqa: E731
    same_tree = canon(tree_g) == canon(tree)
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
    k, n_f, d = 16, plan.n_f, 3
    per = 2.0 * n_f * k ** 3 + 8.0 * (n_f ** 2 * k ** 2 + n_f ** 3 * k)
    flops = per * (plan.form_leaf.size + plan.eval_leaf.size) + 2.0 * d * k ** (d + 1) * plan.d_tgt.size
    ach = flops / (float(np.mean(ms)) * 1e-3) / 1e12
    t0 = time.perf_counter()
    u = pv.fgt_box(tree, vals, 1e-4, 1e-10)
    e2e = time.perf_counter() - t0
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
            "roofline": {"bound": "tensor", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                         "frac": ach / fp64_peak, "alg_per_launch": flops,
                         "accounting": "algorithmic FP64 flops of the whole transform (leaf->PW, "
                                       "PW->grid, direct tables) over its device time",
                         "peak_source": FP64_SRC},
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
    ap.add_argument("--config", type=int, default=5, choices=[2, 3, 5],
                    help="headline point configuration (BASELINE configs[4] = config 5)")
    ap.add_argument("--n", type=int, default=0, help="override N=M (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the config 2/3/4 secondary lines")
    args = ap.parse_args()
    if args.impl == "reference":
        res = run_reference(args)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup()
    res = run_ours(args, world, rank, local)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
