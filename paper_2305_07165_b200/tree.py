"""GPU-built level-restricted point tree (Alg 1) with the reference's data layout.

`build_point_tree` mirrors /root/reference/pkg/src/fgt/tree.py:259-344 (same
arguments, same return tuple (tree, partition, l_c, R), same ValueErrors) but the
construction runs in libfgtcuda.so (Morton codes + radix sort + parallel balance and
dense-fix rounds).  Box ids are canonical (level-major, Morton order within a level)
instead of the reference's creation order; the box set, parent/leaf relations,
per-leaf ascending index lists and subtree point counts are bit-identical.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .planewave import clamp_tolerance, cutoff_factor, cutoff_level


@dataclass
class Tree:
    """Adaptive 2^d-tree (fields of reference tree.Tree, tree.py:53-115)."""

    dim: int
    root_center: np.ndarray
    root_side: float
    periodic: bool
    level: np.ndarray
    parent: np.ndarray
    children: np.ndarray
    coords: np.ndarray
    is_leaf: np.ndarray
    _level_maps: list = field(default=None, repr=False)

    @property
    def n_boxes(self):
        return self.level.shape[0]

    @property
    def n_levels(self):
        return int(self.level.max()) + 1

    @property
    def root_low(self):
        return self.root_center - 0.5 * self.root_side

    def side(self, level):
        return self.root_side / 2 ** np.asarray(level)

    def centers(self, ids=slice(None)):
        lv = self.level[ids]
        s = self.root_side / 2.0 ** lv
        return self.root_low + (self.coords[ids] + 0.5) * s[..., None]

    def boxes_at_level(self, l):
        return np.nonzero(self.level == l)[0]

    def leaves(self):
        return np.nonzero(self.is_leaf)[0]

    def level_map(self, l):
        if self._level_maps is None:
            maps = [dict() for _ in range(self.n_levels)]
            for b in range(self.n_boxes):
                maps[self.level[b]][tuple(self.coords[b])] = b
            self._level_maps = maps
        return self._level_maps[l] if l < len(self._level_maps) else {}

    def find_covering(self, l, coords):
        c = np.asarray(coords)
        for lv in range(l, -1, -1):
            b = self.level_map(lv).get(tuple(c))
            if b is not None:
                return b
            c = c >> 1
        raise RuntimeError("tree has no root covering the query cell")


@dataclass
class PointPartition:
    """Box-sorted view of the sources and targets (reference tree.py:246-256)."""

    src_perm: np.ndarray
    tgt_perm: np.ndarray
    src_start: np.ndarray
    src_count: np.ndarray
    tgt_start: np.ndarray
    tgt_count: np.ndarray
    n_points: np.ndarray


def tree_params(dim, n_s, delta, epsilon, periodic):
    """Fill the C tree parameters; returns (FgtTreeParams, l_c_periodic, R_periodic).

    periodic = 2 selects the root Fourier-series regime (one box: the unit cell)."""
    if n_s < 1:
        raise ValueError("n_s must be >= 1")
    D0 = cutoff_factor(clamp_tolerance(epsilon))
    tp = _lib.FgtTreeParams()
    tp.dim = dim
    tp.periodic = int(periodic)
    tp.n_s = int(n_s)
    tp.D0 = float(D0)
    tp.delta = float(delta)
    l_c, R = (cutoff_level(delta, epsilon, 1.0, kind="density") if periodic else (0, 2.0 * D0))
    tp.l_c_periodic = int(l_c)
    return tp, l_c, R


class DeviceTree:
    """Owning handle of a tree resident on the GPU (fgt_tree*)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            _lib.load().fgt_tree_free(h)

    @property
    def handle(self):
        return self._h

    def info(self):
        inf = _lib.FgtTreeInfo()
        _lib.check(_lib.load().fgt_tree_get_info(self._h, ctypes.byref(inf)))
        return inf

    def to_host(self):
        """(Tree, PointPartition) on the host."""
        inf = self.info()
        nb, d = inf.n_boxes, inf.dim
        i64 = lambda *s: np.empty(s, dtype=np.int64)  # noqa: E731
        level, parent, children, coords = i64(nb), i64(nb), i64(nb, 2 ** d), i64(nb, d)
        is_leaf = np.empty(nb, dtype=np.uint8)
        src_perm, tgt_perm = i64(inf.n_sources), i64(inf.n_targets)
        ss, sc, ts, tc, npt = i64(nb), i64(nb), i64(nb), i64(nb), i64(nb)
        P = _lib.ptr
        _lib.check(_lib.load().fgt_tree_copy_out(
            self._h, P(level), P(parent), P(children), P(coords), P(is_leaf), P(src_perm),
            P(tgt_perm), P(ss), P(sc), P(ts), P(tc), P(npt)))
        tree = Tree(dim=d, root_center=np.array(inf.root_center[:d]), root_side=inf.root_side,
                    periodic=bool(inf.periodic), level=level, parent=parent, children=children,
                    coords=coords, is_leaf=is_leaf.astype(bool))
        part = PointPartition(src_perm=src_perm, tgt_perm=tgt_perm, src_start=ss, src_count=sc,
                              tgt_start=ts, tgt_count=tc, n_points=npt)
        return tree, part

    def lists(self):
        """Target-centric interaction lists (P entries, D entries) as host arrays."""
        lib = _lib.load()
        li = _lib.FgtListInfo()
        _lib.check(lib.fgt_tree_lists(self._h, ctypes.byref(li)))
        d = self.info().dim
        np_, nd_ = li.n_p_entries, li.n_d_entries
        arrs = [np.empty(np_, np.int64), np.empty(np_, np.int64), np.empty((np_, d), np.int64),
                np.empty(nd_, np.int64), np.empty(nd_, np.int64), np.empty((nd_, d), np.int64)]
        _lib.check(lib.fgt_tree_copy_lists(self._h, *[_lib.ptr(a) for a in arrs]))
        return {"P": tuple(arrs[:3]), "D": tuple(arrs[3:]), "info": li}


def _to_device(a):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    return t.to("cuda", non_blocking=False)


def build_device_tree(sources, targets, n_s, delta, epsilon, periodic=False):
    """Build on the GPU; returns (DeviceTree, l_c_hint, R). Inputs are host arrays."""
    import torch
    sources = np.atleast_2d(np.asarray(sources, dtype=float))
    targets = np.atleast_2d(np.asarray(targets, dtype=float))
    if sources.size == 0 and targets.size == 0:
        raise ValueError("need at least one source or target")
    dim = sources.shape[1] if sources.size else targets.shape[1]
    tp, l_c, R = tree_params(dim, n_s, delta, epsilon, periodic)
    ds, dt = _to_device(sources.reshape(-1, dim)), _to_device(targets.reshape(-1, dim))
    h = ctypes.c_void_p()
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.load().fgt_tree_build_dev(
        ctypes.c_void_p(ds.data_ptr()), ds.shape[0], ctypes.c_void_p(dt.data_ptr()), dt.shape[0],
        ctypes.byref(tp), ctypes.c_void_p(stream), ctypes.byref(h)))
    return DeviceTree(h), R


def build_point_tree(sources, targets, n_s, delta, epsilon, periodic=False):
    """Alg 1 on the GPU; returns (tree, partition, l_c, R) like the reference."""
    dt, R = build_device_tree(sources, targets, n_s, delta, epsilon, periodic)
    tree, part = dt.to_host()
    return tree, part, int(dt.info().l_c), R
