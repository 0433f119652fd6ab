"""Continuous (box) FGT on the GPU: Alg 3 density tree (host, or decided on the device),
Alg 4 in CUDA, Alg 5 from retained incoming expansions, Alg 6, interp_at.

Public entry points mirror the reference / SPEC:
  * `build_density_tree(density, dim, k, epsilon, periodic=False, l_max=30,
    refill="evaluate", root_center=None, root_side=1.0)` -> (tree, values, coeffs),
    the contract of /root/reference/pkg/src/fgt/tree.py:394-461 (sigma is a user
    callable, so Alg 3 is driven from the host; boxes are created in the reference's order;
    device="cuda" moves the node generation, sigma, the tail tests and the balance sweeps
    to the GPU);
  * `fgt_box(tree, values, delta, epsilon, boundary="free")` -> {leaf: u (k,)*d}
    (SPEC.md:512-516): the level tables (J/I moments, poly1d.py:129-210) and schedules are
    built here, then one C call (`fgt_box`, include/fgt_cuda.h) runs leaf->PW, merge,
    gather, push, PW->grid and the direct near field on the GPU.
Conventions (signs, lambda = 2 sqrt(delta)/L, pre-multiplied weights) are the ones
SURVEY.md §3(D) verified against quadrature.
"""

import ctypes

from types import SimpleNamespace

import numpy as np
from scipy.special import spherical_jn

from . import _lib
from .planewave import PERIODIC_IMAGE_DELTA, clamp_tolerance, cutoff_level, periodic_params, pw_params
from .tree import Tree

MAX_LEVEL = 30


# ------------------------------------------------------------------ 1-D polynomial tools
def legendre_values(n_max, x):
    """P_0..P_n_max at x (three-term recurrence)."""
    x = np.asarray(x, dtype=float)
    out = np.empty((n_max + 1,) + x.shape)
    out[0] = 1.0
    if n_max:
        out[1] = x
    for n in range(1, n_max):
        out[n + 1] = ((2 * n + 1) * x * out[n] - n * out[n - 1]) / (n + 1)
    return out


class LegendreBasis:
    """k Gauss-Legendre nodes/weights on [-1, 1] and the value <-> coefficient maps."""

    def __init__(self, k):
        if not 2 <= k <= 24:
            raise ValueError(f"polynomial order k={k} outside supported range [2, 24]")
        self.k = k
        self.nodes, self.weights = np.polynomial.legendre.leggauss(k)
        P = legendre_values(k - 1, self.nodes)
        self.val_to_pol = ((2 * np.arange(k) + 1) / 2.0)[:, None] * self.weights[None, :] * P
        self.pol_to_val = P.T.copy()


def apply_per_axis(mat, tensor, dim):
    out = tensor
    for ax in range(dim):
        out = np.moveaxis(np.tensordot(mat, out, axes=([1], [ax])), 0, ax)
    return np.ascontiguousarray(out)


def tail_error(c):
    k, d = c.shape[0], c.ndim
    if d == 1:
        tail = c[k - 2:]
    else:
        idx = np.indices((k,) * d).astype(float)
        tail = c[(idx ** 2).sum(axis=0) >= k * k]
    return float(np.sqrt(np.mean(np.abs(tail) ** 2))) if tail.size else 0.0


def gauss_moment_J(lam, n_max, t):
    """J_lam[P_n](t) = int_{-1}^1 exp(-((t-x)/lam)^2) P_n(x) dx by composite Gauss-Legendre
    quadrature over the support [t-9.5 lam, t+9.5 lam] clipped to [-1, 1]."""
    t = np.atleast_1d(np.asarray(t, dtype=float))
    lo = np.maximum(-1.0, t - 9.5 * lam)
    hi = np.minimum(1.0, t + 9.5 * lam)
    xs, ws = np.polynomial.legendre.leggauss(40)
    out = np.zeros((n_max + 1,) + t.shape)
    panels = 8
    for p in range(panels):
        a = lo + (hi - lo) * (p / panels)
        b = lo + (hi - lo) * ((p + 1) / panels)
        half = 0.5 * np.maximum(b - a, 0.0)
        X = (0.5 * (a + b))[..., None] + half[..., None] * xs
        g = np.exp(-((t[..., None] - X) / lam) ** 2) * (half[..., None] * ws)
        out += np.einsum("n...q,...q->n...", legendre_values(n_max, X), g)
    return out


def fourier_moment_I(n_max, t):
    """I[P_n](t) = int_{-1}^1 exp(i t x) P_n(x) dx = 2 i^n j_n(t)."""
    t = np.atleast_1d(np.asarray(t, dtype=float))
    n = np.arange(n_max + 1)
    jn = spherical_jn(n[:, None], t.ravel()[None, :]).reshape((n_max + 1,) + t.shape)
    return 2.0 * (1j ** n).reshape((-1,) + (1,) * t.ndim) * jn


# ------------------------------------------------------------------ Alg 3
class _Builder:
    """Mutable 2^d-tree in the reference's creation order (children of box b at level l+1
    get consecutive ids; child c has axis-k bit (c >> k) & 1)."""

    def __init__(self, dim, rc, rs, periodic):
        self.dim, self.rc, self.rs, self.periodic = dim, np.asarray(rc, float), float(rs), periodic
        self.level, self.parent, self.kids = [0], [-1], [None]
        self.coords = [np.zeros(dim, np.int64)]
        self.index = [{(0,) * dim: 0}]
        self.bits = np.array([[(c >> a) & 1 for a in range(dim)] for c in range(2 ** dim)])
        g = np.stack(np.meshgrid(*([np.arange(-1, 2)] * dim), indexing="ij"), -1).reshape(-1, dim)
        self.offs = [o for o in g if o.any()]

    def leaf(self, b):
        return self.kids[b] is None

    def center(self, b):
        s = self.rs / 2 ** self.level[b]
        return self.rc - 0.5 * self.rs + (self.coords[b] + 0.5) * s

    def split(self, b):
        l = self.level[b] + 1
        if l > MAX_LEVEL:
            raise RuntimeError(f"refinement beyond maximum level {MAX_LEVEL}")
        if len(self.index) <= l:
            self.index.append({})
        first = len(self.level)
        for c in range(2 ** self.dim):
            g = 2 * self.coords[b] + self.bits[c]
            self.level.append(l)
            self.parent.append(b)
            self.kids.append(None)
            self.coords.append(g)
            self.index[l][tuple(g)] = first + c
        self.kids[b] = list(range(first, first + 2 ** self.dim))
        return self.kids[b]

    def covering(self, l, cell):
        c = np.asarray(cell)
        for lv in range(min(l, len(self.index) - 1), -1, -1):
            b = self.index[lv].get(tuple(c))
            if b is not None:
                return b
            c = c >> 1
        raise RuntimeError("no covering box")

    def _cover_t(self, l, c):
        for lv in range(min(l, len(self.index) - 1), -1, -1):
            b = self.index[lv].get(c)
            if b is not None:
                return b
            c = tuple(x >> 1 for x in c)
        raise RuntimeError("no covering box")

    def balance(self, on_split):
        # same LIFO sweep as the reference builder, on plain-Python tuples
        offs = [tuple(int(x) for x in o) for o in self.offs]
        stack = [b for b in range(len(self.level)) if self.leaf(b)]
        while stack:
            b = stack.pop()
            if not self.leaf(b) or self.level[b] < 2:
                continue
            l, again = self.level[b], False
            n_side = 1 << l
            g = tuple(self.coords[b].tolist())
            for o in offs:
                n = tuple(gi + oi for gi, oi in zip(g, o))
                if self.periodic:
                    n = tuple(x - (x // n_side) * n_side for x in n)
                elif not all(0 <= x < n_side for x in n):
                    continue
                nb = self._cover_t(l, n)
                if self.leaf(nb) and l - self.level[nb] >= 2:
                    kids = self.split(nb)
                    on_split(nb, kids)
                    stack.extend(kids)
                    again = True
            if again:
                stack.append(b)

    def finalize(self):
        nb = len(self.level)
        children = np.full((nb, 2 ** self.dim), -1, np.int64)
        for b, k in enumerate(self.kids):
            if k is not None:
                children[b] = k
        return Tree(dim=self.dim, root_center=self.rc, root_side=self.rs, periodic=self.periodic,
                    level=np.asarray(self.level, np.int64), parent=np.asarray(self.parent, np.int64),
                    children=children, coords=np.asarray(self.coords, np.int64).reshape(nb, self.dim),
                    is_leaf=children[:, 0] < 0)


def leaf_grid(tree, box, basis):
    """Tensor-product Legendre nodes of a box, shape (k,)*d + (d,)."""
    c = tree.centers(box)
    s = float(tree.side(tree.level[box]))
    axes = [c[i] + 0.5 * s * basis.nodes for i in range(tree.dim)]
    return np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)


def build_density_tree(density, dim, k, epsilon, periodic=False, l_max=MAX_LEVEL,
                       refill="evaluate", root_center=None, root_side=1.0, device=None):
    """Resolve sigma on a level-restricted tree (Alg 3); returns (tree, values, coeffs).

    device="cuda": Alg 3 on the GPU (_build_density_tree_device): sigma is a torch function
    evaluated on device-generated grid nodes, the tail test and the level-restriction
    sweeps are CUDA kernels, and the leaf grids stay in HBM until the tree is final.  Same
    box set and leaf grids as the host path; boxes created by the balance are numbered in
    sweep order instead of the reference's LIFO order."""
    if refill != "evaluate":
        # the reference's interpolation refill evaluates at local*0.5 (tree.py:482) and is
        # wrong by O(1); only re-evaluation is supported
        raise ValueError("only refill='evaluate' is supported")
    rc = np.zeros(dim) if root_center is None else np.asarray(root_center, float)
    eps = clamp_tolerance(epsilon)
    basis = LegendreBasis(k)
    if device is not None:
        return _build_density_tree_device(density, dim, k, eps, periodic, l_max, rc, float(root_side),
                                          basis, device)
    B = _Builder(dim, rc, root_side, periodic)
    values, coeffs = {}, {}
    wt = basis.weights
    for _ in range(dim - 1):
        wt = np.multiply.outer(wt, basis.weights)

    def nodes_of(b):
        c = B.center(b)
        s = B.rs / 2 ** B.level[b]
        axes = [c[i] + 0.5 * s * basis.nodes for i in range(dim)]
        return np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)

    def sample_many(boxes):
        # one density call for a whole batch of boxes (sigma acts pointwise, so the values
        # equal per-box calls); coefficients per box as the reference computes them
        if not boxes:
            return
        pts = np.stack([nodes_of(b) for b in boxes])
        if device is None:
            vs = np.asarray(density(pts), float)
        else:
            import torch
            vs = density(torch.from_numpy(pts).to(device)).double().cpu().numpy()
        for b, v in zip(boxes, vs):
            values[b] = v
            coeffs[b] = apply_per_axis(basis.val_to_pol, v, dim)

    def sample(b):
        sample_many([b])

    def sigma_norm():
        tot = 0.0
        for b, v in values.items():
            if B.leaf(b):
                s = B.rs / 2 ** B.level[b]
                tot += (s / 2.0) ** dim * float(np.sum(wt * v * v))
        return np.sqrt(tot) / root_side ** (dim / 2.0)

    sample(0)
    frontier = [0]
    for l in range(l_max + 1):
        nrm = max(sigma_norm(), 1e-300)
        split = [b for b in frontier if tail_error(coeffs[b]) > eps * nrm]
        if not split:
            break
        if l == l_max:
            raise RuntimeError(f"density not resolved at maximum refinement level {l_max}")
        frontier = []
        for b in split:
            frontier.extend(B.split(b))
        sample_many(frontier)
    # balance decisions use only geometry: sample the boxes it creates in one batch
    created = []
    B.balance(lambda parent, kids: created.extend(kids))
    sample_many(created)
    tree = B.finalize()
    leaves = np.nonzero(tree.is_leaf)[0]
    return tree, {b: values[b] for b in leaves}, {b: coeffs[b] for b in leaves}


def _build_density_tree_device(density, dim, k, eps, periodic, l_max, rc, rs, basis, device):
    """Alg 3 with every per-grid decision on the GPU (reference tree.py:394-461).

    Per refinement level: one kernel writes the k^d Gauss-Legendre nodes of the frontier
    boxes (fgt_box_nodes_dev, coordinates rounded like the host expressions), sigma (a torch
    function) is evaluated on them, and one kernel per box turns the values into Legendre
    coefficients and returns the tail estimate and the weighted square sum
    (fgt_box_tail_dev); only those two numbers per box cross PCIe.  The level restriction
    runs as flag sweeps over the sorted (level, Morton) keys (fgt_box_balance_flags) until
    no leaf is flagged; the boxes it creates are sampled in one batch per sweep."""
    import torch
    lib = _lib.load()
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError("the device density-tree build needs a CUDA device")
    nc, kd = 1 << dim, k ** dim
    bits = np.array([[(c >> a) & 1 for a in range(dim)] for c in range(nc)], np.int64)
    low = np.zeros(3)
    low[:dim] = rc - 0.5 * rs
    nodes_h = np.ascontiguousarray(basis.nodes)
    v2p_h = np.ascontiguousarray(basis.val_to_pol)
    w_h = np.ascontiguousarray(basis.weights)
    level = np.zeros(1, np.int32)
    coords = np.zeros((1, dim), np.int64)
    parent = np.full(1, -1, np.int64)
    first_child = np.full(1, -1, np.int64)
    tail = np.zeros(0)
    wsq = np.zeros(0)
    chunks = []  # device tensors (n, k^d) in box-id order

    def sample(lv, cd):
        n = lv.shape[0]
        with torch.cuda.device(dev):
            stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            pts = torch.empty((n,) + (k,) * dim + (dim,), dtype=torch.float64, device=dev)
            _lib.check(lib.fgt_box_nodes_dev(_lib.ptr(np.ascontiguousarray(lv)), _lib.ptr(np.ascontiguousarray(cd)),
                                             n, dim, k, _lib.ptr(nodes_h), _lib.ptr(low), rs,
                                             ctypes.c_void_p(pts.data_ptr()), stream))
            v = density(pts).to(torch.float64).reshape(n, kd).contiguous()
            out = torch.empty((2, n), dtype=torch.float64, device=dev)
            _lib.check(lib.fgt_box_tail_dev(ctypes.c_void_p(v.data_ptr()), n, dim, k, _lib.ptr(v2p_h),
                                            _lib.ptr(w_h), ctypes.c_void_p(out[0].data_ptr()),
                                            ctypes.c_void_p(out[1].data_ptr()), stream))
            tw = out.cpu().numpy()
        chunks.append(v)
        return tw[0], tw[1]

    def split(ids):
        nonlocal level, coords, parent, first_child
        nb = level.shape[0]
        ids = np.asarray(ids, np.int64)
        first_child[ids] = nb + nc * np.arange(ids.size)
        lv = np.repeat(level[ids] + 1, nc).astype(np.int32)
        if lv.size and int(lv.max()) > MAX_LEVEL:
            raise RuntimeError(f"refinement beyond maximum level {MAX_LEVEL}")
        cd = (2 * coords[ids][:, None, :] + bits[None, :, :]).reshape(-1, dim)
        level = np.concatenate([level, lv])
        coords = np.concatenate([coords, cd])
        parent = np.concatenate([parent, np.repeat(ids, nc)])
        first_child = np.concatenate([first_child, np.full(lv.size, -1, np.int64)])
        return np.arange(nb, nb + lv.size), lv, cd

    def grow(tw):
        nonlocal tail, wsq
        tail = np.concatenate([tail, tw[0]])
        wsq = np.concatenate([wsq, tw[1]])

    grow(sample(level, coords))
    frontier = np.zeros(1, np.int64)
    for l in range(l_max + 1):
        leaf = first_child < 0
        nrm = np.sqrt(np.sum((0.5 * rs / 2.0 ** level[leaf]) ** dim * wsq[leaf])) / rs ** (dim / 2.0)
        nrm = max(float(nrm), 1e-300)
        marks = frontier[tail[frontier] > eps * nrm]
        if marks.size == 0:
            break
        if l == l_max:
            raise RuntimeError(f"density not resolved at maximum refinement level {l_max}")
        frontier, lv, cd = split(marks)
        grow(sample(lv, cd))
    while True:
        n = level.shape[0]
        flags = np.zeros(n, np.uint8)
        leaf8 = np.ascontiguousarray((first_child < 0).astype(np.uint8))
        _lib.check(lib.fgt_box_balance_flags(_lib.ptr(level), _lib.ptr(np.ascontiguousarray(coords)),
                                             _lib.ptr(leaf8), n, dim, int(bool(periodic)), _lib.ptr(flags)))
        marks = np.nonzero(flags)[0]
        if marks.size == 0:
            break
        _, lv, cd = split(marks)
        grow(sample(lv, cd))
    n = level.shape[0]
    children = np.where(first_child[:, None] >= 0, first_child[:, None] + np.arange(nc)[None, :], -1)
    tree = Tree(dim=dim, root_center=rc, root_side=rs, periodic=periodic, level=level.astype(np.int64),
                parent=parent, children=children, coords=coords, is_leaf=first_child < 0)
    leaves = np.nonzero(tree.is_leaf)[0]
    allv = torch.cat(chunks) if len(chunks) > 1 else chunks[0]
    V = allv[torch.from_numpy(leaves).to(dev)].cpu().numpy().reshape((leaves.size,) + (k,) * dim)
    C = V
    for ax in range(dim):
        C = np.moveaxis(np.tensordot(basis.val_to_pol, C, axes=([1], [ax + 1])), 0, ax + 1)
    return tree, {int(b): V[i] for i, b in enumerate(leaves)}, {int(b): C[i] for i, b in enumerate(leaves)}


# ------------------------------------------------------------------ Alg 4 plan
FINE = [(-0.75, 0.5), (-0.25, 0.5), (0.25, 0.5), (0.75, 0.5)]
COARSE = [(-1.5, 2.0), (-0.5, 2.0), (0.5, 2.0), (1.5, 2.0)]
COLL = [(-1.0, 1.0), (0.0, 1.0), (1.0, 1.0)]
OFFSETS = FINE + COARSE + COLL  # the 11 per-axis offsets s_1..s_11


class BoxPlan:
    """Host half of Alg 4: flags, lists, tables and shift schedules for one tree."""

    def __init__(self, tree, delta, epsilon, k, periodic):
        if not delta > 0:
            raise ValueError("delta must be positive")
        d = tree.dim
        self.dim, self.k = d, k
        eps = clamp_tolerance(epsilon)
        self.l_c, R = cutoff_level(delta, eps, tree.root_side, kind="density")
        # periodic with cutoff level <= 1: the root Fourier-series regime
        # -- the unit cell is the one plane-wave box, k_n = 2 pi n, |n| <= n_p, weights
        # sqrt(pi delta) exp(-(pi sqrt(delta) n)^2), every leaf merges into it, no near field
        self.root_series = bool(periodic) and not (delta < PERIODIC_IMAGE_DELTA and self.l_c >= 2)
        if self.root_series:
            ser = periodic_params(eps, delta)
            self.l_c = 0
            self.pw = SimpleNamespace(n_f=2 * ser.n_p + 1, h=2.0 * np.pi * np.sqrt(delta),
                                      weights_1d=ser.coeffs)
            periodic = False  # the series carries every image
        else:
            self.pw = pw_params(float(epsilon), delta, R=R, dim=d)
        n_f = self.n_f = self.pw.n_f
        basis = self.basis = LegendreBasis(k)
        nb = tree.n_boxes
        l_c = self.l_c
        lmax = int(tree.level.max())
        self.n_levels = max(lmax, l_c) + 1
        leaves = np.nonzero(tree.is_leaf)[0]
        self.leaves = leaves
        leaf_slot = np.full(nb, -1, np.int64)
        leaf_slot[leaves] = np.arange(leaves.size)
        # plain-Python views of the tree (per-element numpy indexing dominated this plan)
        lev = tree.level.tolist()
        crd = [tuple(c) for c in tree.coords.tolist()]
        isleaf = tree.is_leaf.tolist()
        kids = tree.children.tolist()
        key = {(lev[b],) + crd[b]: b for b in range(nb)}
        self._plan_views = (lev, crd, isleaf, kids, key)
        km = (np.arange(n_f) - n_f // 2) * self.pw.h / np.sqrt(delta)
        side = tree.root_side / 2.0 ** np.arange(self.n_levels)
        offs = [tuple(o) for o in
                np.stack(np.meshgrid(*([np.arange(-1, 2)] * d), indexing="ij"), -1).reshape(-1, d).tolist()]
        zero = (0,) * d

        def covering(l, cell):
            c = cell
            for lv in range(l, -1, -1):
                b = key.get((lv,) + c)
                if b is not None:
                    return b
                c = tuple(x >> 1 for x in c)
            raise RuntimeError("no covering box")

        def neighbour_cells(b, with_self=True):
            n_side = 1 << lev[b]
            g = crd[b]
            for o in offs:
                if not with_self and o == zero:
                    continue
                n = tuple(gi + oi for gi, oi in zip(g, o))
                if periodic:
                    v = tuple(x // n_side for x in n)
                    yield tuple(x - vi * n_side for x, vi in zip(n, v)), v
                elif all(0 <= x < n_side for x in n):
                    yield n, zero

        # f flags (Definition fflagdef): level > l_c, or level l_c with a subdivided colleague
        f = tree.level > l_c
        coll = {}
        for b in np.nonzero(tree.level == l_c)[0].tolist():
            # colleagues that exist at l_c (a coarser covering leaf interacts directly)
            lst = [(key[kk], v) for n, v in neighbour_cells(b) if (kk := (l_c,) + n) in key]
            coll[b] = lst
            f[b] = any(not isleaf[S] for S, _ in lst) or self.root_series
        pw_slot = np.full(nb, -1, np.int64)
        pw_slot[f] = np.arange(int(f.sum()))
        self.n_pw = int(f.sum())
        self.pw_slot, self.leaf_slot = pw_slot, leaf_slot
        fl = f.tolist()
        slot = pw_slot.tolist()

        # ---- phase rows: out2in (3) at l_c, then c2p (2) and p2c (2) per child level
        rows = [np.exp(1j * km * o * side[l_c]) for o in (-1, 0, 1)]
        c2p_row, p2c_row = {}, {}
        for l in range(1, self.n_levels):
            for sgn in (0, 1):
                s = (2 * sgn - 1) * 0.5 * side[l]
                c2p_row[(l, sgn)] = len(rows)
                rows.append(np.exp(-1j * km * s))
                p2c_row[(l, sgn)] = len(rows)
                rows.append(np.exp(1j * km * s))
        self.rows = np.ascontiguousarray(np.array(rows, dtype=np.complex128))
        self.p2c_row = p2c_row

        # ---- shift stages: merge (deepest first), gather at l_c, push (shallowest first)
        stage_off, stage_kind = [0], []
        dst, dst_acc, dst_off, ent_src, ent_rows = [], [], [0], [], []

        def add_dst(t, entries, acc=0):
            dst.append(slot[t])
            dst_acc.append(acc)
            for s_, r in entries:
                ent_src.append(slot[s_])
                ent_rows.append(r)
            dst_off.append(len(ent_src))

        def end_stage(kind):
            if len(dst) > stage_off[-1]:
                stage_off.append(len(dst))
                stage_kind.append(kind)

        def child_rows(b, c, table, l1):
            return [table[(l1, ci - 2 * bi)] for ci, bi in zip(crd[c], crd[b])]

        for l in range(lmax - 1, l_c - 1, -1):
            for b in np.nonzero((tree.level == l) & ~tree.is_leaf)[0].tolist():
                add_dst(b, [(c, child_rows(b, c, c2p_row, l + 1)) for c in kids[b]])
            end_stage(0)
        n_gpairs = 0
        side_c = 1 << l_c
        for T, lst in coll.items():
            if not fl[T]:
                continue
            ents = []
            for S, v in lst:
                if fl[S] and (self.root_series or not (isleaf[T] and isleaf[S])):
                    # o = coords_T - coords_S - v 2^l_c, in {-1, 0, 1}
                    ents.append((S, [t - s_ - vi * side_c + 1 for t, s_, vi in zip(crd[T], crd[S], v)]))
            n_gpairs += len(ents)
            add_dst(T, ents)
        end_stage(1)
        self.n_gather_pairs = n_gpairs
        for l in range(l_c, lmax):
            for b in np.nonzero((tree.level == l) & ~tree.is_leaf & f)[0].tolist():
                for c in kids[b]:
                    add_dst(c, [(b, child_rows(b, c, p2c_row, l + 1))])
            end_stage(2)
        self.stage_off = np.array(stage_off, np.int64)
        self.stage_kind = np.array(stage_kind, np.int64)
        self.dst = np.array(dst, np.int64)
        self.dst_acc = np.array(dst_acc, np.int64)
        self.dst_off = np.array(dst_off, np.int64)
        self.ent_src = np.array(ent_src, np.int64)
        self.ent_rows = np.array(ent_rows, np.int64).reshape(-1, d)

        # ---- leaf -> PW and PW -> grid
        fl = leaves[f[leaves]]
        self.form_leaf = leaf_slot[fl]
        self.form_pw = pw_slot[fl]
        self.form_level = tree.level[fl].astype(np.int64)
        self.eval_leaf, self.eval_pw, self.eval_level = self.form_leaf, self.form_pw, self.form_level
        val2pw = np.zeros((self.n_levels, n_f, k), np.complex128)
        pw2val = np.zeros((self.n_levels, k, n_f), np.complex128)
        m = np.arange(n_f) - n_f // 2
        for l in set(self.form_level.tolist()):
            L = side[l]
            I = fourier_moment_I(k - 1, L * m * self.pw.h / (2 * np.sqrt(delta)))  # (k, n_f)
            val2pw[l] = ((L / 2.0) * self.pw.weights_1d[:, None] * np.conj(I).T) @ basis.val_to_pol
            pw2val[l] = np.exp(1j * np.outer(0.5 * L * basis.nodes, km))
        self.val2pw = np.ascontiguousarray(val2pw)
        self.pw2val = np.ascontiguousarray(pw2val)

        # ---- direct: touching leaf pairs with both leaves at level <= l_c (D-list)
        pairs = []
        for T in (leaves[tree.level[leaves] <= l_c].tolist() if not self.root_series else []):
            lt = lev[T]
            side_t = 1 << lt
            gT = crd[T]
            seen = set()
            for n, v in neighbour_cells(T):
                S = covering(lt, n)
                if isleaf[S]:
                    cands = [S]
                else:
                    cands = [c for c in kids[S]
                             if all(2 * gt - 1 <= gc + 2 * vi * side_t <= 2 * gt + 2
                                    for gc, vi, gt in zip(crd[c], v, gT))]
                for S2 in cands:
                    kk = (S2,) + v
                    if kk in seen or not isleaf[S2] or lev[S2] > l_c:
                        continue
                    seen.add(kk)
                    pairs.append((T, S2, v))
        ctr = tree.centers()
        used_levels = sorted({lev[S] for _, S, _ in pairs})
        tab_id = {}
        tabs = []
        for l in used_levels:
            L = side[l]
            lam = 2 * np.sqrt(delta) / L
            for j, (o, r) in enumerate(OFFSETS):
                Jm = gauss_moment_J(lam, k - 1, 2 * o + r * basis.nodes)  # (k deg, k tgt)
                tab_id[(l, j)] = len(tabs)
                tabs.append(((L / 2.0) * Jm.T) @ basis.val_to_pol)
        self.dtab = np.ascontiguousarray(np.array(tabs, np.float64).reshape(-1, k, k))
        look = {(o, r): j for j, (o, r) in enumerate(OFFSETS)}
        ctr_l = ctr.tolist()
        side_l = side.tolist()
        rs = float(tree.root_side)
        d_t, d_s, d_tab = [], [], []
        # per target leaf: (source leaf slot, image shift) -- what Alg 5 hands to new children
        self.d_sources = {}
        for T, S, v in pairs:
            self.d_sources.setdefault(T, []).append((int(leaf_slot[S]), lev[S], crd[S], v))
        for T, S, v in sorted(pairs, key=lambda p: leaf_slot[p[0]]):
            ls = lev[S]
            Ls, Lt = side_l[ls], side_l[lev[T]]
            ratio = Lt / Ls
            cT, cS = ctr_l[T], ctr_l[S]
            d_tab.append([tab_id[(ls, look[((cT[ax] - cS[ax] - v[ax] * rs) / Ls, ratio)])] for ax in range(d)])
            d_t.append(int(leaf_slot[T]))
            d_s.append(int(leaf_slot[S]))
        self.d_tgt = np.array(d_t, np.int64)
        self.d_src = np.array(d_s, np.int64)
        self.d_tab = np.array(d_tab, np.int64).reshape(-1, d)

    def cstruct(self):
        """The fgt_box_plan C struct (arrays kept alive by self)."""
        return _plan_cstruct(self)


def _plan_cstruct(self):
        """fgt_box_plan from any object with BoxPlan's array attributes (BoxPlan, _RefinePlan)."""
        P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if a.dtype != np.int64 else \
            a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))  # noqa: E731
        self._keep = [np.ascontiguousarray(a) for a in (
            self.val2pw.view(np.float64), self.pw2val.view(np.float64), self.rows.view(np.float64),
            self.dtab)]
        s = _lib.FgtBoxPlan()
        s.dim, s.k, s.n_f, s.n_levels, s.l_c = self.dim, self.k, self.n_f, self.n_levels, self.l_c
        s.n_leaves, s.n_pw = self.leaves.size, self.n_pw
        s.val2pw, s.pw2val = P(self._keep[0]), P(self._keep[1])
        s.n_rows, s.rows = self.rows.shape[0], P(self._keep[2])
        s.n_tables, s.dtab = self.dtab.shape[0], P(self._keep[3])
        s.n_form, s.form_leaf, s.form_pw, s.form_level = (
            self.form_leaf.size, P(self.form_leaf), P(self.form_pw), P(self.form_level))
        s.n_stages, s.n_dst, s.n_entries = self.stage_kind.size, self.dst.size, self.ent_src.size
        s.stage_off, s.stage_kind = P(self.stage_off), P(self.stage_kind)
        s.dst, s.dst_acc, s.dst_off = P(self.dst), P(self.dst_acc), P(self.dst_off)
        self._ent_rows = np.ascontiguousarray(self.ent_rows)
        s.ent_src, s.ent_rows = P(self.ent_src), P(self._ent_rows)
        s.n_eval, s.eval_leaf, s.eval_pw, s.eval_level = (
            self.eval_leaf.size, P(self.eval_leaf), P(self.eval_pw), P(self.eval_level))
        self._d_tab = np.ascontiguousarray(self.d_tab)
        s.n_dpairs, s.d_tgt, s.d_src, s.d_tab = self.d_tgt.size, P(self.d_tgt), P(self.d_src), P(self._d_tab)
        return s


def _host_buffer(shape):
    """float64 host array in page-locked memory when a GPU is present (torch's caching host
    allocator): the leaf grids cross PCIe at link speed instead of through the driver's
    pageable staging."""
    try:
        import torch
        if torch.cuda.is_available():
            return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    except ImportError:
        pass
    return np.empty(shape, dtype=np.float64)


def _stack_values(tree, values, k, pinned=False):
    leaves = np.nonzero(tree.is_leaf)[0]
    shape = (len(leaves),) + (k,) * tree.dim
    V = _host_buffer(shape) if pinned else np.empty(shape, dtype=np.float64)
    np.stack([np.asarray(values[b], float).reshape((k,) * tree.dim) for b in leaves], out=V)
    return leaves, V


class RetainedTransform:
    """Device state kept after fgt_box(..., retain=True): psi of every f = 1 box and the
    density's leaf grids (fgt_box_state), with the plan and tree they belong to.  Input of
    refine_output (Alg 5, "incoming expansions retained for f=1 boxes")."""

    def __init__(self, handle, plan, tree, leaves, delta, epsilon, boundary):
        self.handle, self.plan, self.tree, self.leaves = handle, plan, tree, leaves
        self.delta, self.epsilon, self.boundary = delta, epsilon, boundary
        self.n_pw = plan.n_pw

    def free(self):
        if self.handle is not None:
            _lib.load().fgt_box_state_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # interpreter shutdown
            pass


def fgt_box(tree, values, delta, epsilon, boundary="free", return_times=False, plan=None, retain=False):
    """u = int exp(-|x-y|^2/delta) sigma(y) dy on every leaf grid; {leaf: (k,)*d array}.
    retain=True also returns a RetainedTransform (the last element of the result)."""
    if boundary not in ("free", "periodic"):
        raise ValueError(f"unknown boundary {boundary!r}")
    if bool(tree.periodic) != (boundary == "periodic"):
        raise ValueError("tree periodicity does not match boundary")
    some = next(iter(values.values()))
    k = np.asarray(some).shape[0]
    plan = plan or BoxPlan(tree, delta, epsilon, k, boundary == "periodic")
    leaves, V = _stack_values(tree, values, k, pinned=True)
    U = _host_buffer(V.shape)
    t = _lib.FgtPhaseTimes()
    cs = plan.cstruct()
    state = None
    if retain:
        handle = ctypes.c_void_p()
        _lib.check(_lib.load().fgt_box_retain(ctypes.byref(cs), _lib.ptr(V), _lib.ptr(U), ctypes.byref(t),
                                              ctypes.byref(handle)))
        state = RetainedTransform(handle, plan, tree, leaves, delta, epsilon, boundary)
    else:
        _lib.check(_lib.load().fgt_box(ctypes.byref(cs), _lib.ptr(V), _lib.ptr(U), ctypes.byref(t)))
    out = {int(b): U[i] for i, b in enumerate(leaves)}
    res = (out, t.as_dict()) if return_times else (out,)
    if retain:
        res = res + (state,)
    return res if len(res) > 1 else res[0]


def fgt_box_device(plan, values_dev, out_dev=None, return_times=False):
    """Box FGT on torch CUDA tensors (n_leaves, k^d) already resident in HBM."""
    import torch
    if out_dev is None:
        out_dev = torch.empty_like(values_dev)
    t = _lib.FgtPhaseTimes()
    cs = plan.cstruct()
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.load().fgt_box_dev(ctypes.byref(cs), ctypes.c_void_p(values_dev.data_ptr()),
                                       ctypes.c_void_p(out_dev.data_ptr()), ctypes.c_void_p(stream),
                                       ctypes.byref(t)))
    return (out_dev, t.as_dict()) if return_times else out_dev


def interp_at(tree, potentials, targets):
    """Values of a box-FGT output at arbitrary points (per-target leaf
    lookup + tensor Legendre evaluation of the leaf's coefficient tensor; PAPER.md section
    4.2 "simply use polynomial interpolation").  potentials: {leaf: (k,)*d grid values}
    as returned by fgt_box; targets (n, d) inside the root box (wrapped if periodic).
    Runs on the GPU (fgt_box_interp); out-of-domain points give nan."""
    d = tree.dim
    leaves = np.nonzero(tree.is_leaf)[0]
    k = np.asarray(potentials[int(leaves[0])]).shape[0]
    V = np.stack([np.asarray(potentials[int(b)], float).reshape((k,) * d) for b in leaves])
    basis = LegendreBasis(k)
    C = V
    for ax in range(d):  # values -> Legendre coefficients, axis by axis, all leaves at once
        C = np.moveaxis(np.tensordot(basis.val_to_pol, C, axes=([1], [ax + 1])), 0, ax + 1)
    C = np.ascontiguousarray(C.reshape(len(leaves), -1))
    lev = np.ascontiguousarray(tree.level[leaves], dtype=np.int32)
    crd = np.ascontiguousarray(tree.coords[leaves], dtype=np.int64)
    x = np.ascontiguousarray(np.atleast_2d(np.asarray(targets, dtype=np.float64)).reshape(-1, d))
    t = _lib.FgtInterpTree()
    t.dim, t.k, t.periodic, t.n_leaves = d, k, int(bool(tree.periodic)), len(leaves)
    t.level = lev.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    t.coords = crd.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    t.coeffs = C.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    low = np.zeros(3)
    low[:d] = tree.root_low
    t.root_low = (ctypes.c_double * 3)(*low)
    t.root_side = float(tree.root_side)
    out = np.empty(x.shape[0])
    _lib.check(_lib.load().fgt_box_interp(ctypes.byref(t), _lib.ptr(x), x.shape[0], _lib.ptr(out)))
    return out



def _coarsen_output_device(tree, potentials, epsilon):
    """Alg 6 with the per-grid work on the GPU: per level, the k^d nodes of every candidate
    parent (all children leaves) are evaluated through the current tree's leaf interpolants
    (`fgt_box_interp`: the deepest leaf holding a node is the child the host sweep picks,
    Gauss-Legendre nodes being interior) and tested by the tail kernel (`fgt_box_tail`); the
    host only edits the tree.  Same merges as the host sweep."""
    d = tree.dim
    k = np.asarray(next(iter(potentials.values()))).shape[0]
    basis = LegendreBasis(k)
    pots = {int(b): np.asarray(v, float).reshape((k,) * d) for b, v in potentials.items()}
    is_leaf = tree.is_leaf.copy()
    alive = np.ones(tree.n_boxes, bool)
    for lev in range(int(tree.level.max()) - 1, -1, -1):
        cand = [int(b) for b in np.nonzero((tree.level == lev) & ~is_leaf & alive)[0]
                if all(is_leaf[c] for c in tree.children[b])]
        if not cand:
            continue
        cur = Tree(dim=d, root_center=tree.root_center, root_side=tree.root_side, periodic=tree.periodic,
                   level=tree.level, parent=tree.parent, children=tree.children, coords=tree.coords,
                   is_leaf=is_leaf & alive)
        nodes = np.concatenate([leaf_grid(tree, b, basis).reshape(-1, d) for b in cand])
        V = interp_at(cur, pots, nodes).reshape((len(cand),) + (k,) * d)
        te = tail_errors(V, d, k)
        for i, b in enumerate(cand):
            if te[i] <= epsilon:
                pots[b] = V[i]
                is_leaf[b] = True
                for c in tree.children[b]:
                    alive[c] = False
                    pots.pop(int(c), None)
    return _renumber_alive(tree, is_leaf, alive, pots)


def coarsen_output(tree, potentials, epsilon, device=None):
    """Alg 6: bottom-up, a non-leaf box whose
    children are all leaves gets the potential at its own k^d grid by evaluating whichever
    child holds each node; if that grid's Legendre tail error (Eq. funerr, tail_error) is
    <= epsilon the children are deleted and the box becomes a leaf.  Returns (tree,
    potentials) with boxes renumbered (level-restriction is not re-imposed).
    device="cuda": the interpolation and the tail tests run on the GPU, one batch per level
    (_coarsen_output_device); None: host numpy."""
    if device is not None:
        return _coarsen_output_device(tree, potentials, epsilon)
    d = tree.dim
    k = np.asarray(next(iter(potentials.values()))).shape[0]
    basis = LegendreBasis(k)
    pots = {int(b): np.asarray(v, float).reshape((k,) * d) for b, v in potentials.items()}
    is_leaf = tree.is_leaf.copy()
    alive = np.ones(tree.n_boxes, bool)
    nc = 1 << d
    bits = np.array([[(c >> a) & 1 for a in range(d)] for c in range(nc)])
    for lev in range(int(tree.level.max()) - 1, -1, -1):
        for b in np.nonzero((tree.level == lev) & ~is_leaf & alive)[0]:
            ch = tree.children[b]
            if not all(is_leaf[c] for c in ch):
                continue
            # parent nodes -> containing child (node > 0 along an axis -> upper child) and
            # that child's local coordinate 2 x - (+-1)
            g = np.stack(np.meshgrid(*([basis.nodes] * d), indexing="ij"), -1).reshape(-1, d)
            up = (g > 0).astype(int)
            loc = 2.0 * g - np.where(up == 1, 1.0, -1.0)
            vals = np.empty(g.shape[0])
            for c in range(nc):
                sel = np.all(up == bits[c], axis=1)
                if not sel.any():
                    continue
                child = int(ch[c])
                coef = apply_per_axis(basis.val_to_pol, pots[child], d)
                P = [legendre_values(k - 1, loc[sel, a]) for a in range(d)]  # (k, m)
                if d == 1:
                    vals[sel] = coef @ P[0]
                elif d == 2:
                    vals[sel] = np.einsum("ab,am,bm->m", coef, P[0], P[1])
                else:
                    vals[sel] = np.einsum("abc,am,bm,cm->m", coef, P[0], P[1], P[2])
            V = vals.reshape((k,) * d)
            if tail_error(apply_per_axis(basis.val_to_pol, V, d)) <= epsilon:
                pots[int(b)] = V
                is_leaf[b] = True
                for c in ch:
                    alive[c] = False
                    pots.pop(int(c), None)
    return _renumber_alive(tree, is_leaf, alive, pots)


def _renumber_alive(tree, is_leaf, alive, pots):
    # renumber the surviving boxes (creation order kept)
    d = tree.dim
    keep = np.nonzero(alive)[0]
    new_id = np.full(tree.n_boxes, -1, np.int64)
    new_id[keep] = np.arange(keep.size)
    children = tree.children[keep].copy()
    children[is_leaf[keep]] = -1
    children = np.where(children >= 0, new_id[np.maximum(children, 0)], -1)
    parent = np.where(tree.parent[keep] >= 0, new_id[np.maximum(tree.parent[keep], 0)], -1)
    out = Tree(dim=d, root_center=tree.root_center, root_side=tree.root_side, periodic=tree.periodic,
               level=tree.level[keep].copy(), parent=parent, children=children,
               coords=tree.coords[keep].copy(), is_leaf=is_leaf[keep].copy())
    return out, {int(new_id[b]): v for b, v in pots.items() if alive[b] and is_leaf[b]}


def tail_errors(grids, dim, k, return_wsq=False):
    """Eq. (funerr) tail estimates of a stack of leaf grids (n, k^d), on the GPU
    (fgt_box_tail; the reference's tail_error, poly1d.py:116-126, per grid); with
    return_wsq also the Gauss-Legendre weighted square sums sum_i w_i v_i^2."""
    G = np.ascontiguousarray(np.asarray(grids, float).reshape(-1, k ** dim))
    basis = LegendreBasis(k)
    out = np.empty(G.shape[0])
    wsq = np.empty(G.shape[0]) if return_wsq else None
    _lib.check(_lib.load().fgt_box_tail(_lib.ptr(G), G.shape[0], dim, k,
                                        _lib.ptr(np.ascontiguousarray(basis.val_to_pol)),
                                        _lib.ptr(np.ascontiguousarray(basis.weights)), _lib.ptr(out),
                                        _lib.ptr(wsq)))
    return (out, wsq) if return_wsq else out


def grid_norm(tree, grids, k):
    """||f||_2 of a piecewise polynomial given by its leaf grids, normalised by the root
    volume (the sigma norm of Alg 3, tree.py:417-428): sqrt(sum_leaves (side/2)^d sum_i w_i
    f_i^2 / side_0^d)."""
    leaves = sorted(grids)
    _, wsq = tail_errors(np.stack([np.asarray(grids[b], float) for b in leaves]), tree.dim, k, return_wsq=True)
    half = 0.5 * tree.root_side / 2.0 ** tree.level[leaves]
    return float(np.sqrt(np.sum(half ** tree.dim * wsq)) / tree.root_side ** (tree.dim / 2.0))


def direct_table_key(lt, gt, ls, gs, v):
    """Per-axis centre offset (c_T - c_S - v L_0) / L_S and side ratio L_T / L_S of a target box
    (level lt, integer coords gt) and a source box (ls, gs) under image shift v: the key of
    the T_pol2pot table of the pair (J_lam[P_n](2 o + r xi); any level
    difference, Alg 5 Remark).  Dyadic numbers from integer box coordinates: exact in floating
    point, so equal pairs share a table."""
    r = 2.0 ** (ls - lt)
    return [(2 * int(gt[ax]) + 1) * 0.5 * r - (2 * int(gs[ax]) + 1) * 0.5 - int(v[ax]) * float(1 << ls)
            for ax in range(len(gs))], r


class _RefinePlan:
    """fgt_box_plan for one Alg 5 sweep: pushes into new plane-wave slots, PW -> grid on the
    new leaves, direct tables for arbitrary (offset, side ratio) pairs (Alg 5 Remark)."""

    def __init__(self, base, n_levels):
        self.dim, self.k, self.n_f, self.l_c = base.dim, base.k, base.n_f, base.l_c
        self.n_levels = n_levels
        self.rows = base.rows
        self.val2pw = np.zeros((n_levels, base.n_f, base.k), np.complex128)
        e = np.zeros(0, np.int64)
        self.form_leaf = self.form_pw = self.form_level = e


def refine_output(tree, values, potentials=None, delta=None, epsilon=None, boundary="free",
                  max_rounds=30, state=None, return_stats=False, relative=False):
    """Alg 5: refine the output tree until every
    leaf's potential passes the tail test (Eq. funerr) at epsilon, evaluating each new child
    from the RETAINED incoming expansion of its parent.

    state = the RetainedTransform of fgt_box(tree, values, ..., retain=True) (computed here
    when absent).  A sweep tests the leaves created by the previous one (all leaves at first;
    tail kernel on the GPU), splits the failing ones and, in ONE device call
    (fgt_box_refine): psi_child = T_p2c psi_parent when f(parent) = 1, u_child = T_pw2pot
    psi_child, plus the direct part from the parent's D-list sources (the
    parent's list is a safe superset) through T_pol2pot tables built for the actual centre
    offset and side ratio of each (source, child) pair -- the extended tables of the Alg 5
    Remark, keyed by (source level, offset / L_S, L_T / L_S), exact dyadic numbers.  The
    density of a split leaf goes to its children by exact polynomial refill (sigma is
    unchanged; sources of direct pairs stay the ORIGINAL leaf grids, which represent the
    same polynomial).  Refinement never goes deeper than the input tree (Alg 5 Remark).
    relative=True tests e(B) > epsilon ||u||_2 (the normalisation Alg 3 uses for sigma,
    PAPER.md:965) instead of Alg 5's literal e(B) > epsilon.
    The final level-restriction sweep ("if desired, rebalance") evaluates the boxes it
    creates the same way.  Returns (tree, values, potentials, n_sweeps[, stats])."""
    d = tree.dim
    k = np.asarray(next(iter(values.values()))).shape[0]
    basis = LegendreBasis(k)
    own_state = state is None
    if own_state:
        if delta is None or epsilon is None:
            raise ValueError("delta and epsilon are needed to compute the retained transform")
        potentials, state = fgt_box(tree, values, delta, epsilon, boundary, retain=True)
    elif potentials is None:
        raise ValueError("potentials of the retained transform are required")
    if state.handle is None:
        raise ValueError("the retained transform was freed")
    delta, eps_pw = state.delta, state.epsilon
    epsilon = eps_pw if epsilon is None else epsilon
    plan = state.plan
    lmax = int(tree.level.max())
    n_levels = plan.n_levels
    rs = float(tree.root_side)
    side = rs / 2.0 ** np.arange(n_levels)
    n_f = plan.n_f
    km = (np.arange(n_f) - n_f // 2) * plan.pw.h / np.sqrt(delta)
    pw2val = np.zeros((n_levels, k, n_f), np.complex128)
    for l in range(n_levels):
        pw2val[l] = np.exp(1j * np.outer(0.5 * side[l] * basis.nodes, km))
    p2c_row = plan.p2c_row  # (child level, child bit) -> phase row of the base plan
    # child refill operators: P(t)^T with t the child's nodes in the parent's coordinates
    M = [legendre_values(k - 1, 0.5 * basis.nodes + (0.5 if bit else -0.5)).T for bit in (0, 1)]
    B = _Builder(d, tree.root_center, tree.root_side, bool(tree.periodic))
    B.level, B.parent = tree.level.tolist(), tree.parent.tolist()
    B.coords = [np.asarray(c, np.int64) for c in tree.coords]
    B.kids = [None if tree.is_leaf[b] else tree.children[b].tolist() for b in range(tree.n_boxes)]
    B.index = [dict() for _ in range(lmax + 1)]
    for b in range(tree.n_boxes):
        B.index[tree.level[b]][tuple(tree.coords[b])] = b
    vals = {int(b): np.asarray(v, float).reshape((k,) * d) for b, v in values.items()}
    pots = {int(b): np.asarray(v, float).reshape((k,) * d) for b, v in potentials.items()}
    pw = {int(b): int(plan.pw_slot[b]) for b in np.nonzero(tree.is_leaf)[0]}
    dsrc = {int(b): plan.d_sources.get(int(b), []) for b in pw}
    n_pw = state.n_pw
    stats = {"added": 0, "balance_added": 0, "pushes": 0, "direct_pairs": 0, "tables": 0}
    tab_cache = {}

    def refill(b, kids):
        coef = apply_per_axis(basis.val_to_pol, vals.pop(b), d)
        for c, kid in enumerate(kids):
            out = coef
            for ax in range(d):
                out = np.moveaxis(np.tensordot(M[(c >> ax) & 1], out, axes=([1], [ax])), 0, ax)
            vals[kid] = np.ascontiguousarray(out)

    class Sweep:
        """Children to evaluate in one fgt_box_refine call."""

        def __init__(self):
            self.kids, self.push, self.pairs = [], [], []  # (kid), (level, dst, src, rows), (row, S, tabs)
            self.tabs, self.tab_id = [], {}

        def table(self, ls, o, r):
            key = (ls, o, r)
            t = self.tab_id.get(key)
            if t is None:
                mat = tab_cache.get(key)
                if mat is None:
                    Ls = side[ls]
                    Jm = gauss_moment_J(2 * np.sqrt(delta) / Ls, k - 1, 2 * o + r * basis.nodes)
                    mat = tab_cache[key] = ((Ls / 2.0) * Jm.T) @ basis.val_to_pol
                    stats["tables"] += 1
                t = self.tab_id[key] = len(self.tabs)
                self.tabs.append(mat)
            return t

        def add(self, b, kids):
            nonlocal n_pw
            refill(b, kids)
            pots.pop(b, None)
            for kid in kids:
                lk = B.level[kid]
                g = B.coords[kid]
                row = len(self.kids)
                self.kids.append(kid)
                if pw[b] >= 0:
                    pw[kid] = n_pw
                    n_pw += 1
                    self.push.append((lk, pw[kid], pw[b],
                                      [p2c_row[(lk, int(gc - 2 * gb))] for gc, gb in zip(g, B.coords[b])]))
                else:
                    pw[kid] = -1
                dsrc[kid] = dsrc[b]
                for S, ls, gs, v in dsrc[b]:
                    offs, r = direct_table_key(lk, g, ls, gs, v)
                    tabs = [self.table(ls, o, r) for o in offs]
                    self.pairs.append((row, S, tabs))

        def run(self):
            if not self.kids:
                return
            rp = _RefinePlan(plan, n_levels)
            rp.leaves = np.arange(len(self.kids))
            rp.n_pw = n_pw
            rp.pw2val = pw2val
            rp.dtab = (np.ascontiguousarray(np.array(self.tabs, np.float64).reshape(-1, k, k))
                       if self.tabs else np.zeros((0, k, k)))
            push = sorted(self.push, key=lambda e: e[0])  # parents before children
            stage_off, stage_kind, last = [0], [], None
            for i, e in enumerate(push):
                if last is not None and (e[0] != last or i - stage_off[-1] >= 65535):
                    stage_off.append(i)
                    stage_kind.append(2)
                last = e[0]
            if push:
                stage_off.append(len(push))
                stage_kind.append(2)
            rp.stage_off = np.array(stage_off, np.int64)
            rp.stage_kind = np.array(stage_kind, np.int64)
            rp.dst = np.array([e[1] for e in push], np.int64)
            rp.dst_acc = np.zeros(len(push), np.int64)
            rp.dst_off = np.arange(len(push) + 1, dtype=np.int64)
            rp.ent_src = np.array([e[2] for e in push], np.int64)
            rp.ent_rows = np.array([e[3] for e in push], np.int64).reshape(-1, d)
            ev = [(i, pw[kid], B.level[kid]) for i, kid in enumerate(self.kids) if pw[kid] >= 0]
            rp.eval_leaf = np.array([e[0] for e in ev], np.int64)
            rp.eval_pw = np.array([e[1] for e in ev], np.int64)
            rp.eval_level = np.array([e[2] for e in ev], np.int64)
            rp.d_tgt = np.array([p[0] for p in self.pairs], np.int64)
            rp.d_src = np.array([p[1] for p in self.pairs], np.int64)
            rp.d_tab = np.array([p[2] for p in self.pairs], np.int64).reshape(-1, d)
            U = np.empty((len(self.kids),) + (k,) * d)
            cs = _plan_cstruct(rp)
            _lib.check(_lib.load().fgt_box_refine(state.handle, ctypes.byref(cs), _lib.ptr(U), None))
            state.n_pw = n_pw
            for i, kid in enumerate(self.kids):
                pots[kid] = U[i]
            stats["pushes"] += len(push)
            stats["direct_pairs"] += len(self.pairs)

    sweeps = 0
    fresh = sorted(pots)
    if relative:
        epsilon = epsilon * max(grid_norm(tree, pots, k), 1e-300)
    stats["threshold"] = epsilon
    try:
        while fresh and sweeps < max_rounds:
            cand = [b for b in fresh if B.level[b] < lmax]
            if not cand:
                break
            te = tail_errors(np.stack([pots[b] for b in cand]), d, k)
            marks = [b for b, e in zip(cand, te) if e > epsilon]
            if not marks:
                break
            sw = Sweep()
            for b in marks:
                sw.add(b, B.split(b))
            sw.run()
            stats["added"] += len(sw.kids)
            fresh = sw.kids
            sweeps += 1
        sw = Sweep()
        B.balance(sw.add)
        sw.run()
        stats["balance_added"] = len(sw.kids)
    finally:
        if own_state:
            state.free()
    cur = B.finalize()
    leaf_ids = np.nonzero(cur.is_leaf)[0].tolist()
    out = (cur, {b: vals[b] for b in leaf_ids}, {b: pots[b] for b in leaf_ids}, sweeps)
    return out + (stats,) if return_stats else out
