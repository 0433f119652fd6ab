"""Discrete plane-wave FGT (Alg 2 of arXiv 2305.07165) on the GPU.

Entry point `fgt_points(sources, charges, targets, delta, epsilon, n_s, boundary)`
keeps the contract of the reference's (specified, unshipped) point_fgt module,
/root/reference/SPEC.md:408-412 and :149-163:

    u_i = sum_j exp(-||x_i - y_j||^2 / delta) q_j,   relative l2 error <= ~10 eps.

Host work is parameter selection only (bit-identical numpy expressions, see
planewave.py); the tree, lists, outgoing expansions, translations, evaluation and
direct sums all run in libfgtcuda.so.  `fgt_points_device` takes torch CUDA tensors
(inputs already resident in HBM) and runs on torch's current stream.
"""

import ctypes

import numpy as np

from . import _lib
from .planewave import (EPS_MAX, EPS_MIN, PERIODIC_IMAGE_DELTA, clamp_tolerance, cutoff_factor,
                        periodic_params, pw_params)
from .tree import tree_params


class FgtParams:
    """Resolved parameters of one transform (tree + plane-wave quadrature)."""

    def __init__(self, dim, delta, epsilon, n_s, periodic, share=(0, 1)):
        if not delta > 0:
            raise ValueError("delta must be positive")
        # the supported tolerance window of planewave.pw_params (planewave.py:80-82), enforced
        # for every boundary; inside it the tree, the near-field cut and the quadrature all use
        # the same clamped value (clamp_tolerance only moves [0.099, 0.1) to 0.099)
        if not (EPS_MIN <= float(epsilon) < EPS_MAX):
            raise ValueError(f"unsupported tolerance {float(epsilon):g}; need 1e-14 <= eps < 0.1")
        eps = clamp_tolerance(epsilon)
        self.tp, self.l_c_periodic, self.R = tree_params(dim, n_s, delta, eps, periodic)
        rank, size = share
        if not 0 <= rank < size:
            raise ValueError(f"bad share {share!r}")
        self.tp.part_rank, self.tp.part_size = int(rank), int(size)
        pw = _lib.FgtPwParams()
        pw.dim = dim
        pw.delta = float(delta)
        self.root_series = bool(periodic) and not (delta < PERIODIC_IMAGE_DELTA and self.l_c_periodic >= 2)
        if self.root_series:
            # l_c <= 1: the periodic Gaussian's Fourier
            # series on the root, k_n = 2 pi n, |n| <= n_p, weights sqrt(pi delta)
            # exp(-(pi sqrt(delta) n)^2).  One box (the unit cell) holds every point; its
            # outgoing expansion is its incoming one; no near field.
            self.series = periodic_params(eps, delta)
            self.tp.periodic = 2
            self.tp.n_s = 0
            self._w = np.ascontiguousarray(self.series.coeffs, dtype=np.float64)
            pw.n_f = 2 * self.series.n_p + 1
            pw.D0 = float(cutoff_factor(eps))
            pw.h = float(2.0 * np.pi * np.sqrt(delta))  # k = h n / sqrt(delta) = 2 pi n
        else:
            # NUFFT/plane-wave rule for the cutoff boxes
            self.pwq = pw_params(float(eps), delta, R=self.R, dim=dim)
            self._w = np.ascontiguousarray(self.pwq.weights_1d, dtype=np.float64)
            pw.n_f = self.pwq.n_f
            pw.D0 = float(self.pwq.D0)
            pw.h = float(self.pwq.h)
        pw.weights_1d = self._w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        self.pw = pw


_PARAMS_CACHE = {}


def _params(dim, delta, epsilon, n_s, periodic, share):
    """FgtParams memoised on its arguments (the host quadrature and cutoff-level set-up
    is ~0.05 ms; repeated transforms with the same parameters reuse it read-only)."""
    key = (int(dim), float(delta), float(epsilon), int(n_s), bool(periodic), tuple(share))
    p = _PARAMS_CACHE.get(key)
    if p is None:
        p = FgtParams(dim, delta, epsilon, n_s, periodic, share)
        if len(_PARAMS_CACHE) > 64:
            _PARAMS_CACHE.clear()
        _PARAMS_CACHE[key] = p
    return p


def _prep(sources, charges, targets, periodic):
    src = np.atleast_2d(np.asarray(sources, dtype=np.float64))
    tgt = np.atleast_2d(np.asarray(targets, dtype=np.float64))
    q = np.asarray(charges, dtype=np.float64).reshape(-1)
    if src.size == 0 and tgt.size == 0:
        raise ValueError("need at least one source or target")
    dim = src.shape[1] if src.size else tgt.shape[1]
    src = src.reshape(-1, dim)
    tgt = tgt.reshape(-1, dim)
    if q.shape[0] != src.shape[0]:
        raise ValueError("sources/charges length mismatch")
    if periodic:
        # the unit cell is [-1/2, 1/2)^d; wrap points given outside it
        if src.size and (src.min() < -0.5 or src.max() >= 0.5):
            src = src - np.floor(src + 0.5)
        if tgt.size and (tgt.min() < -0.5 or tgt.max() >= 0.5):
            tgt = tgt - np.floor(tgt + 0.5)
    return np.ascontiguousarray(src), np.ascontiguousarray(q), np.ascontiguousarray(tgt), dim


def _boundary(boundary):
    if boundary not in ("free", "periodic"):
        raise ValueError(f"unknown boundary {boundary!r}")
    return boundary == "periodic"


def _host_out(n):
    """Result buffer in page-locked memory (torch's caching host allocator, reused across
    calls): the device->host copy of u runs at link speed instead of through the driver's
    pageable staging.  A plain numpy array backed by the pinned block."""
    import torch

    if torch.cuda.is_available():
        return torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    return np.empty(n, dtype=np.float64)


def fgt_points(sources, charges, targets, delta, epsilon, n_s, boundary="free",
               return_times=False, share=(0, 1), out=None):
    """Potentials u (M,) at the targets; host arrays in, host array out.

    share=(rank, size) evaluates only this rank's cost-balanced range of target leaves
    (other targets get 0); summing the outputs of all ranks gives the full transform.
    out: optional caller-owned (M,) float64 C-contiguous host array that receives u
    (overwritten, not accumulated) and is returned; page-locked memory makes the
    device->host copy run at link speed.
    """
    periodic = _boundary(boundary)
    src, q, tgt, dim = _prep(sources, charges, targets, periodic)
    prm = _params(dim, delta, epsilon, n_s, periodic, share)
    if out is None:
        u = _host_out(tgt.shape[0])
    else:
        if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.shape == (tgt.shape[0],)
                and out.flags.c_contiguous and out.flags.writeable):
            raise ValueError("out must be a writeable C-contiguous float64 array of shape (M,)")
        u = out
    times = _lib.FgtPhaseTimes()
    P = _lib.ptr
    _lib.check(_lib.load().fgt_points(P(src), src.shape[0], P(q), P(tgt), tgt.shape[0],
                                      ctypes.byref(prm.tp), ctypes.byref(prm.pw), P(u),
                                      ctypes.byref(times)))
    return (u, times.as_dict()) if return_times else u


def fgt_points_device(sources, charges, targets, delta, epsilon, n_s, boundary="free",
                      out=None, params=None, return_times=False, share=(0, 1)):
    """Same transform on torch CUDA float64 tensors (resident in HBM)."""
    import torch
    periodic = _boundary(boundary)
    for name, t in (("sources", sources), ("charges", charges), ("targets", targets)):
        if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous CUDA float64 tensor")
    dim = sources.shape[1] if sources.dim() == 2 else targets.shape[1]
    prm = params or _params(dim, delta, epsilon, n_s, periodic, share)
    nt = targets.shape[0]
    if out is None:
        out = torch.empty(nt, dtype=torch.float64, device=targets.device)
    times = _lib.FgtPhaseTimes()
    stream = torch.cuda.current_stream().cuda_stream
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    _lib.check(_lib.load().fgt_points_dev(vp(sources), sources.shape[0], vp(charges), vp(targets),
                                          nt, ctypes.byref(prm.tp), ctypes.byref(prm.pw),
                                          vp(out), ctypes.c_void_p(stream), ctypes.byref(times)))
    return (out, times.as_dict()) if return_times else out


class TorchExchange:
    """Halo exchange of outgoing expansions over torch.distributed (NCCL over NVLink):
    one all-to-all of the packed slots (SURVEY.md section 8(e) exchange 1)."""

    def __init__(self, group=None):
        self.group = group

    def __call__(self, send, recv, send_counts, recv_counts, slot):
        import torch.distributed as dist
        dist.all_to_all_single(recv, send, [int(c) * slot for c in recv_counts],
                               [int(c) * slot for c in send_counts], group=self.group)

    def assemble(self, u):
        """u of the whole transform on every rank (SURVEY.md section 8(e) exchange 3): each
        target is owned by exactly one rank and the others hold an exact 0.0 there, so a sum
        over ranks reproduces the single-GPU result bit for bit (one NCCL all-reduce)."""
        import torch.distributed as dist
        dist.all_reduce(u, op=dist.ReduceOp.SUM, group=self.group)
        return u


def fgt_points_exchange_begin(sources, charges, targets, delta, epsilon, n_s, boundary="free",
                              share=(0, 1)):
    """Phase 1 of a multi-GPU transform with the expansion halo exchanged instead of
    recomputed: returns a PointsRun (tree, lists, this rank's owned expansions formed)."""
    import torch
    periodic = _boundary(boundary)
    for name, t in (("sources", sources), ("charges", charges), ("targets", targets)):
        if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous CUDA float64 tensor")
    dim = sources.shape[1] if sources.dim() == 2 else targets.shape[1]
    prm = FgtParams(dim, delta, epsilon, n_s, periodic, share)
    return PointsRun(prm, sources, charges, targets)


class PointsRun:
    """An fgt_points_run handle: begin -> (pack / exchange / unpack) -> finish."""

    def __init__(self, prm, sources, charges, targets):
        import torch
        self.prm = prm
        self.world = prm.tp.part_size
        self.nt = targets.shape[0]
        self.device = targets.device
        self.stream = torch.cuda.current_stream().cuda_stream
        h = ctypes.c_void_p()
        vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _lib.check(_lib.load().fgt_points_begin(vp(sources), sources.shape[0], vp(charges), vp(targets),
                                                self.nt, ctypes.byref(prm.tp), ctypes.byref(prm.pw),
                                                ctypes.c_void_p(self.stream), ctypes.byref(h)))
        self._h = h
        self._keep = (sources, charges, targets)
        sc = (ctypes.c_int64 * self.world)()
        rc = (ctypes.c_int64 * self.world)()
        slot = ctypes.c_int64()
        _lib.check(_lib.load().fgt_points_exchange_counts(h, sc, rc, ctypes.byref(slot)))
        self.send_counts, self.recv_counts, self.slot = list(sc), list(rc), slot.value

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            _lib.load().fgt_points_run_free(h)

    def pack(self):
        import torch
        buf = torch.empty(sum(self.send_counts) * self.slot, dtype=torch.float64, device=self.device)
        _lib.check(_lib.load().fgt_points_pack(self._h, ctypes.c_void_p(buf.data_ptr())))
        return buf

    def unpack(self, buf):
        _lib.check(_lib.load().fgt_points_unpack(self._h, ctypes.c_void_p(buf.data_ptr())))

    def exchange(self, exchanger):
        import torch
        send = self.pack()
        recv = torch.empty(sum(self.recv_counts) * self.slot, dtype=torch.float64, device=self.device)
        exchanger(send, recv, self.send_counts, self.recv_counts, self.slot)
        self.unpack(recv)

    def finish(self, out=None, return_times=False):
        import torch
        if out is None:
            out = torch.empty(self.nt, dtype=torch.float64, device=self.device)
        times = _lib.FgtPhaseTimes()
        _lib.check(_lib.load().fgt_points_finish(self._h, ctypes.c_void_p(out.data_ptr()), ctypes.byref(times)))
        return (out, times.as_dict()) if return_times else out

