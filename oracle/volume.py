"""Oracle: continuous (box) FGT -- Alg 3 density tree + Alg 4.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
  * `legendre`, `vals_to_coeffs`, `tail_error`: poly1d.py:26-126
  * `gauss_J`: J_lam[P_n](t) = int_{-1}^{1} exp(-((t-x)/lam)^2) P_n(x) dx (poly1d.py:175-195),
    here by composite Gauss-Legendre on the clipped support (the reference switches to
    the same clipped quadrature outside its recurrence window, poly1d.py:161-172)
  * `fourier_I`: I[P_n](t) = 2 i^n j_n(t) (poly1d.py:198-210)
  * `density_tree`: tree.build_density_tree (tree.py:394-461), refill="evaluate"
  * `fgt_box`: Alg 4 with the conventions SURVEY.md §3(D) verified against quadrature:
    phi_m = w_m (L/2)^d sum_a c_a prod conj(I[P_{a_i}](L m_i h / (2 sqrt(delta)))),
    child->parent exp(-ik.(c_C-c_B)), out->in exp(+ik.(c_T-c_S-v)),
    parent->child exp(+ik.(c_C-c_B)), u = Re sum_m exp(ik.(x-c_B)) psi_m;
    direct (L/2) J_lam[P_n](2(x-c_S)/L), lam = 2 sqrt(delta)/L.
    PW pairs: colleagues at l_c with f=1 on both sides and not both leaves; D pairs:
    touching leaf-leaf pairs at levels <= l_c (incl. self).
"""

import numpy as np
from scipy.special import spherical_jn

from .params import clamp_eps, cut_level, quad
from .point_fgt import neighbour_lists
from .tree import Boxes, offsets


# ------------------------------------------------------------------ 1-D machinery
def legendre(n_max, x):
    """P_0..P_n_max at x: shape (n_max+1,) + x.shape (poly1d.legendre_values :38-47)."""
    x = np.asarray(x, dtype=float)
    P = np.empty((n_max + 1,) + x.shape)
    P[0] = 1.0
    if n_max >= 1:
        P[1] = x
    for n in range(1, n_max):
        P[n + 1] = ((2 * n + 1) * x * P[n] - n * P[n - 1]) / (n + 1)
    return P


class Basis:
    """Gauss-Legendre nodes/weights and the val->pol map (poly1d.LegendreBasis :50-73)."""

    def __init__(self, k):
        self.k = k
        self.nodes, self.weights = np.polynomial.legendre.leggauss(k)
        P = legendre(k - 1, self.nodes)
        self.v2p = ((2 * np.arange(k)[:, None] + 1) / 2.0) * self.weights[None, :] * P
        self.p2v = P.T.copy()


def apply_axes(mats, t):
    """Apply mats[i] (m_i x k) along axis i of tensor t (poly1d._apply_per_axis :76-81)."""
    out = t
    for ax, M in enumerate(mats):
        out = np.moveaxis(np.tensordot(M, out, axes=([1], [ax])), 0, ax)
    return out


def tail_error(c):
    """RMS of the coefficient tail ||alpha||_2 >= k (poly1d.tail_error :100-126)."""
    k, d = c.shape[0], c.ndim
    if d == 1:
        sel = c[k - 2:]
    else:
        g = np.meshgrid(*([np.arange(k)] * d), indexing="ij")
        sel = c[sum(x.astype(float) ** 2 for x in g) >= k * k]
    return float(np.sqrt(np.mean(np.abs(sel) ** 2))) if sel.size else 0.0


def gauss_J(lam, n_max, t):
    """J_lam[P_0..n_max](t), shape (n_max+1,) + t.shape, composite clipped quadrature."""
    t = np.atleast_1d(np.asarray(t, dtype=float))
    lo = np.maximum(-1.0, t - 9.5 * lam)
    hi = np.minimum(1.0, t + 9.5 * lam)
    xs, ws = np.polynomial.legendre.leggauss(48)
    out = np.zeros((n_max + 1,) + t.shape)
    npan = 6
    for p in range(npan):
        a = lo + (hi - lo) * p / npan
        b = lo + (hi - lo) * (p + 1) / npan
        X = 0.5 * (a + b)[..., None] + 0.5 * (b - a)[..., None] * xs
        W = 0.5 * np.maximum(b - a, 0.0)[..., None] * ws
        g = np.exp(-((t[..., None] - X) / lam) ** 2) * W
        out += np.einsum("n...q,...q->n...", legendre(n_max, X), g)
    return out


def fourier_I(n_max, t):
    """I[P_0..n_max](t) = 2 i^n j_n(t), complex, shape (n_max+1,) + t.shape."""
    t = np.atleast_1d(np.asarray(t, dtype=float))
    n = np.arange(n_max + 1)
    jn = spherical_jn(n[:, None], t.ravel()[None, :]).reshape((n_max + 1,) + t.shape)
    return 2.0 * (1j ** n).reshape((-1,) + (1,) * t.ndim) * jn


# ------------------------------------------------------------------ Alg 3
class DensityTree:
    def __init__(self, B, values, basis):
        nb = len(B.level)
        self.dim, self.periodic = B.dim, B.periodic
        self.root_center, self.root_side = B.rc, B.rs
        self.level = np.asarray(B.level, dtype=np.int64)
        self.parent = np.asarray(B.parent, dtype=np.int64)
        self.children = np.full((nb, 2 ** B.dim), -1, dtype=np.int64)
        for b, kk in enumerate(B.kids):
            if kk is not None:
                self.children[b] = kk
        self.coords = np.asarray(B.coords, dtype=np.int64).reshape(nb, B.dim)
        self.is_leaf = self.children[:, 0] < 0
        self.values = {b: values[b] for b in range(nb) if self.is_leaf[b]}
        self.basis = basis

    @property
    def n_boxes(self):
        return self.level.shape[0]

    def centers(self):
        s = self.root_side / 2.0 ** self.level
        return (self.root_center - 0.5 * self.root_side) + (self.coords + 0.5) * s[:, None]

    def side(self, b):
        return self.root_side / 2.0 ** self.level[b]

    def leaf_points(self, b):
        c = self.centers()[b]
        s = self.side(b)
        axes = [c[i] + 0.5 * s * self.basis.nodes for i in range(self.dim)]
        return np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)


def density_tree(density, dim, k, epsilon, periodic=False, l_max=30, root_side=1.0):
    """tree.build_density_tree (tree.py:394-461) with refill='evaluate'."""
    eps = clamp_eps(epsilon)
    basis = Basis(k)
    B = Boxes(dim, np.zeros(dim), root_side, periodic)
    values, coeffs = {}, {}
    wt = basis.weights
    for _ in range(dim - 1):
        wt = np.multiply.outer(wt, basis.weights)

    def sample(b):
        c = B.center(b)
        s = B.rs / 2 ** B.level[b]
        axes = [c[i] + 0.5 * s * basis.nodes for i in range(dim)]
        pts = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)
        v = np.asarray(density(pts), dtype=float)
        values[b] = v
        coeffs[b] = apply_axes([basis.v2p] * dim, v)

    def norm():
        tot = 0.0
        for b, v in values.items():
            if B.leaf(b):
                s = B.rs / 2 ** B.level[b]
                tot += (s / 2.0) ** dim * float(np.sum(wt * v * v))
        return np.sqrt(tot) / root_side ** (dim / 2.0)

    sample(0)
    frontier = [0]
    for l in range(l_max + 1):
        nrm = max(norm(), 1e-300)
        splits = [b for b in frontier if tail_error(coeffs[b]) > eps * nrm]
        if not splits:
            break
        if l == l_max:
            raise RuntimeError("density not resolved at maximum refinement level")
        frontier = []
        for b in splits:
            kids = B.split(b)
            for c in kids:
                sample(c)
            frontier += kids

    def refill(parent, kids):
        for c in kids:
            sample(c)

    B.balance(refill)
    return DensityTree(B, values, basis)


# ------------------------------------------------------------------ Alg 4
def box_lists(tree, l_c):
    """f flags, PW pairs (T, S, v) at l_c and D pairs (T, S, v)."""
    nb = tree.n_boxes
    keymap = {}
    for b in range(nb):
        keymap[(int(tree.level[b]),) + tuple(int(c) for c in tree.coords[b])] = b
    f = np.zeros(nb, dtype=bool)
    f[tree.level > l_c] = True
    colleagues = {}
    for b in np.nonzero(tree.level == l_c)[0]:
        side = 2 ** l_c
        lst = []
        for o in offsets(tree.dim):
            n = tree.coords[b] + o
            if tree.periodic:
                v = n // side
                n = n - v * side
            else:
                if np.any(n < 0) or np.any(n >= side):
                    continue
                v = np.zeros(tree.dim, dtype=np.int64)
            S = keymap.get((l_c,) + tuple(int(c) for c in n))
            if S is not None:
                lst.append((S, v))
        colleagues[b] = lst
        if any(not tree.is_leaf[S] for S, _ in lst):
            f[b] = True
    pw_pairs = []
    for T, lst in colleagues.items():
        if not f[T]:
            continue
        for S, v in lst:
            if f[S] and not (tree.is_leaf[T] and tree.is_leaf[S]):
                pw_pairs.append((T, S, v))
    d_pairs = []
    for T in np.nonzero(tree.is_leaf & (tree.level <= l_c))[0]:
        for S, v in neighbour_lists(tree, T):
            if tree.is_leaf[S] and tree.level[S] <= l_c:
                d_pairs.append((T, S, v))
    return f, pw_pairs, d_pairs


def fgt_box(tree, delta, epsilon, boundary="free"):
    """Potentials u[b] (k^d) on every leaf grid: int exp(-|x-y|^2/delta) sigma(y) dy."""
    d, k, basis = tree.dim, tree.basis.k, tree.basis
    eps = clamp_eps(epsilon)
    l_c, R = cut_level(delta, eps, tree.root_side, kind="density")
    pw = quad(eps, delta, R=R, dim=d)
    m = pw.m
    kf = m * pw.h / np.sqrt(delta)
    ctr = tree.centers()
    f, pw_pairs, d_pairs = box_lists(tree, l_c)
    side = lambda b: tree.side(b)  # noqa: E731
    coeffs = {b: apply_axes([basis.v2p] * d, v) for b, v in tree.values.items()}
    phi, psi = {}, {}
    # leaf -> plane waves (Lemma 3.5, point-FGT sign convention)
    for b in coeffs:
        if f[b]:
            L = side(b)
            A = (L / 2.0) * pw.w1[:, None] * np.conj(fourier_I(k - 1, L * m * pw.h / (2 * np.sqrt(delta)))).T
            phi[b] = apply_axes([A] * d, coeffs[b].astype(complex))
    # merge up (child -> parent), deepest level first
    for l in range(int(tree.level.max()) - 1, l_c - 1, -1):
        for b in np.nonzero((tree.level == l) & ~tree.is_leaf)[0]:
            acc = np.zeros((pw.n_f,) * d, dtype=complex)
            for c in tree.children[b]:
                dv = ctr[c] - ctr[b]
                ph = np.exp(-1j * kf * dv[0])
                for ax in range(1, d):
                    ph = np.multiply.outer(ph, np.exp(-1j * kf * dv[ax]))
                acc += ph * phi[c]
            phi[b] = acc
    # gather at l_c
    for T, S, v in pw_pairs:
        dv = ctr[T] - ctr[S] - v * tree.root_side
        ph = np.exp(1j * kf * dv[0])
        for ax in range(1, d):
            ph = np.multiply.outer(ph, np.exp(1j * kf * dv[ax]))
        psi[T] = psi.get(T, 0) + ph * phi[S]
    # push down
    for l in range(l_c, int(tree.level.max())):
        for b in np.nonzero((tree.level == l) & ~tree.is_leaf)[0]:
            if b not in psi:
                continue
            for c in tree.children[b]:
                dv = ctr[c] - ctr[b]
                ph = np.exp(1j * kf * dv[0])
                for ax in range(1, d):
                    ph = np.multiply.outer(ph, np.exp(1j * kf * dv[ax]))
                psi[c] = ph * psi[b]
    u = {b: np.zeros((k,) * d) for b in coeffs}
    for b in coeffs:
        if b in psi:
            L = side(b)
            E = np.exp(1j * np.outer(0.5 * L * basis.nodes, kf))  # (k, n_f)
            u[b] += np.real(apply_axes([E] * d, psi[b]))
    # direct (Lemma 3.4, lam = 2 sqrt(delta)/L_S)
    for T, S, v in d_pairs:
        Ls, Lt = side(S), side(T)
        lam = 2 * np.sqrt(delta) / Ls
        mats = []
        for ax in range(d):
            off = ctr[T][ax] - ctr[S][ax] - v[ax] * tree.root_side
            tt = 2.0 * (off + 0.5 * Lt * basis.nodes) / Ls
            mats.append((Ls / 2.0) * gauss_J(lam, k - 1, tt).T)  # (k targets, k degrees)
        u[T] += apply_axes(mats, coeffs[S])
    return u


def gaussian_box_convolution(x, delta, centers, widths, amps, lo=-0.5, hi=0.5):
    """Closed form of int_{[lo,hi]^d} exp(-|x-y|^2/delta) sum_i a_i exp(-|y-c_i|^2/w_i^2) dy."""
    from scipy.special import erf
    x = np.asarray(x, dtype=float)
    out = np.zeros(x.shape[:-1])
    for c, w, a in zip(centers, widths, amps):
        term = a * np.ones(x.shape[:-1])
        for ax in range(x.shape[-1]):
            xk = x[..., ax]
            s2 = delta + w * w
            mu = (xk * w * w + c[ax] * delta) / s2
            tau = np.sqrt(delta * w * w / s2)
            term = term * np.exp(-(xk - c[ax]) ** 2 / s2) * (np.sqrt(np.pi) * tau / 2) * (
                erf((hi - mu) / tau) - erf((lo - mu) / tau))
        out += term
    return out
