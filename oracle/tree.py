"""Oracle: level-restricted point tree, Alg 1 (restates /root/reference/pkg/src/fgt/tree.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Follows the reference's
sequential construction order exactly (creation-order box ids, LIFO balance queue),
so box ids as well as the box set match the reference:
  root/l_c (tree.py:275-289), level-synchronous split of boxes with > n_s points
  (:493-502), point redistribution by p >= centre (:478-491), 2:1 balance
  (:378-403), dense-cutoff-leaf fix (:506-523), partition (:533-564).
"""

import numpy as np

from .params import clamp_eps, cut_level, d0_of

NO_IDX = np.zeros(0, dtype=np.int64)


def offsets(dim):
    """tree._offsets (tree.py:236-243): axis 0 slowest, values (-1, 0, 1)."""
    g = np.stack(np.meshgrid(*([np.array([-1, 0, 1])] * dim), indexing="ij"), axis=-1)
    return [row.astype(np.int64) for row in g.reshape(-1, dim)]


class Boxes:
    """Mutable struct-of-lists tree (tree._Builder, tree.py:118-233)."""

    def __init__(self, dim, rc, rs, periodic):
        self.dim, self.rc, self.rs, self.periodic = dim, np.asarray(rc, dtype=float), float(rs), periodic
        self.level, self.parent = [0], [-1]
        self.kids = [None]
        self.coords = [np.zeros(dim, dtype=np.int64)]
        self.at = [{(0,) * dim: 0}]
        self.bits = np.array([[(c >> k) & 1 for k in range(dim)] for c in range(2 ** dim)],
                             dtype=np.int64)
        self.offs = [o for o in offsets(dim) if o.any()]

    def leaf(self, b):
        return self.kids[b] is None

    def center(self, b):
        s = self.rs / 2 ** self.level[b]
        return self.rc - 0.5 * self.rs + (self.coords[b] + 0.5) * s

    def split(self, b):
        l = self.level[b] + 1
        if l > 30:
            raise RuntimeError("refinement beyond maximum level")
        if len(self.at) <= l:
            self.at.append({})
        ids = []
        for c in range(2 ** self.dim):
            g = 2 * self.coords[b] + self.bits[c]
            nid = len(self.level)
            self.level.append(l)
            self.parent.append(b)
            self.kids.append(None)
            self.coords.append(g)
            self.at[l][tuple(g)] = nid
            ids.append(nid)
        self.kids[b] = ids
        return ids

    def covering(self, l, cell):
        c = np.asarray(cell)
        for lv in range(min(l, len(self.at) - 1), -1, -1):
            b = self.at[lv].get(tuple(c))
            if b is not None:
                return b
            c = c >> 1
        raise RuntimeError("no covering box")

    def neighbour_cells(self, b):
        """tree._Builder.neighbor_cells (tree.py:176-193), self excluded."""
        n_side = 2 ** self.level[b]
        out = []
        for o in self.offs:
            n = self.coords[b] + o
            if self.periodic:
                v = n // n_side
                out.append((n - v * n_side, v))
            elif not (np.any(n < 0) or np.any(n >= n_side)):
                out.append((n, np.zeros(self.dim, dtype=np.int64)))
        return out

    def balance(self, on_split):
        """tree._Builder.balance (tree.py:195-220), LIFO over leaves."""
        stack = [b for b in range(len(self.level)) if self.leaf(b)]
        while stack:
            b = stack.pop()
            if not self.leaf(b) or self.level[b] < 2:
                continue
            l = self.level[b]
            redo = False
            for cell, _ in self.neighbour_cells(b):
                nb = self.covering(l, cell)
                if self.leaf(nb) and l - self.level[nb] >= 2:
                    kids = self.split(nb)
                    on_split(nb, kids)
                    stack.extend(kids)
                    redo = True
            if redo:
                stack.append(b)


class OracleTree:
    """Finalised tree + partition (tree.Tree / tree.PointPartition fields)."""

    def __init__(self, B, src_ids, tgt_ids, l_c, R):
        nb = len(B.level)
        self.dim, self.periodic = B.dim, B.periodic
        self.root_center, self.root_side = B.rc, B.rs
        self.level = np.asarray(B.level, dtype=np.int64)
        self.parent = np.asarray(B.parent, dtype=np.int64)
        self.children = np.full((nb, 2 ** B.dim), -1, dtype=np.int64)
        for b, k in enumerate(B.kids):
            if k is not None:
                self.children[b] = k
        self.coords = np.asarray(B.coords, dtype=np.int64).reshape(nb, B.dim)
        self.is_leaf = self.children[:, 0] < 0
        self.l_c, self.R = l_c, R
        # partition (tree._sort_points, tree.py:350-381)
        self.src_start = np.zeros(nb, np.int64)
        self.src_count = np.zeros(nb, np.int64)
        self.tgt_start = np.zeros(nb, np.int64)
        self.tgt_count = np.zeros(nb, np.int64)
        sp, tp = [], []
        s = t = 0
        for b in np.nonzero(self.is_leaf)[0]:
            si, ti = src_ids.get(b, NO_IDX), tgt_ids.get(b, NO_IDX)
            self.src_start[b], self.src_count[b] = s, si.size
            self.tgt_start[b], self.tgt_count[b] = t, ti.size
            s += si.size
            t += ti.size
            sp.append(si)
            tp.append(ti)
        self.src_perm = np.concatenate(sp) if sp else NO_IDX
        self.tgt_perm = np.concatenate(tp) if tp else NO_IDX
        self.n_points = np.zeros(nb, np.int64)
        for b in np.argsort(self.level, kind="stable")[::-1]:
            if self.is_leaf[b]:
                self.n_points[b] = self.src_count[b] + self.tgt_count[b]
            if self.parent[b] >= 0:
                self.n_points[self.parent[b]] += self.n_points[b]

    @property
    def n_boxes(self):
        return self.level.shape[0]

    def centers(self):
        s = self.root_side / 2.0 ** self.level
        return (self.root_center - 0.5 * self.root_side) + (self.coords + 0.5) * s[:, None]


def build(sources, targets, n_s, delta, epsilon, periodic=False):
    """tree.build_point_tree (tree.py:259-344)."""
    sources = np.atleast_2d(np.asarray(sources, dtype=float))
    targets = np.atleast_2d(np.asarray(targets, dtype=float))
    if sources.size == 0 and targets.size == 0:
        raise ValueError("need at least one source or target")
    if n_s < 1:
        raise ValueError("n_s must be >= 1")
    dim = sources.shape[1]
    if periodic:
        rc, rs = np.zeros(dim), 1.0
        l_c, R = cut_level(delta, epsilon, 1.0, kind="density")
    else:
        allp = np.vstack([sources, targets])
        lo, hi = allp.min(axis=0), allp.max(axis=0)
        rc = 0.5 * (lo + hi)
        extent = float((hi - lo).max())
        l_c, R = cut_level(delta, epsilon, extent, kind="point")
        rs = 2 ** l_c * d0_of(clamp_eps(epsilon)) * np.sqrt(delta)
        if rs < extent:
            l_c += 1
            rs *= 2.0
    B = Boxes(dim, rc, rs, periodic)
    ids = ({0: np.arange(sources.shape[0])}, {0: np.arange(targets.shape[0])})

    def count(b):
        return ids[0].get(b, NO_IDX).size + ids[1].get(b, NO_IDX).size

    def move(b, kids):
        cb = B.center(b)
        for store, pts in zip(ids, (sources, targets)):
            idx = store.pop(b, None)
            if idx is None or idx.size == 0:
                for c in kids:
                    store[c] = NO_IDX
                continue
            child = ((pts[idx] >= cb) * (1 << np.arange(dim))).sum(axis=1)
            for c, kid in enumerate(kids):
                store[kid] = idx[child == c]

    level_boxes = [0]
    for _ in range(l_c):
        nxt = []
        for b in level_boxes:
            if count(b) > n_s:
                kids = B.split(b)
                move(b, kids)
                nxt += kids
        level_boxes = nxt
    B.balance(move)
    while True:
        changed = False
        for b in range(len(B.level)):
            if not B.leaf(b) or B.level[b] != l_c or count(b) <= n_s:
                continue
            for cell, _ in B.neighbour_cells(b):
                nb = B.covering(l_c, cell)
                if B.leaf(nb) and B.level[nb] == l_c - 1:
                    move(nb, B.split(nb))
                    changed = True
        if not changed:
            break
        B.balance(move)
    return OracleTree(B, ids[0], ids[1], l_c, R)


def canonical(level, coords, is_leaf, n_points, src_start, src_count, src_perm, tgt_start,
              tgt_count, tgt_perm, parent):
    """Order-independent view of a tree for bit-exact comparison.

    Returns a dict keyed by (level, coords tuple) -> (is_leaf, n_points, parent key,
    tuple(src ids), tuple(tgt ids)).
    """
    keys = [(int(level[b]),) + tuple(int(c) for c in coords[b]) for b in range(len(level))]
    out = {}
    for b, k in enumerate(keys):
        s = tuple(src_perm[src_start[b]:src_start[b] + src_count[b]].tolist()) if is_leaf[b] else ()
        t = tuple(tgt_perm[tgt_start[b]:tgt_start[b] + tgt_count[b]].tolist()) if is_leaf[b] else ()
        pk = keys[parent[b]] if parent[b] >= 0 else None
        out[k] = (bool(is_leaf[b]), int(n_points[b]), pk, s, t)
    return out
