"""Oracle: discrete plane-wave FGT, Alg 2 (contract /root/reference/SPEC.md:361-444).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The reference ships no driver;
this restates Alg 2 on the oracle primitives with the semantics
SURVEY.md §3(B)/§8(c) fixed against exact sums:
  * P-boxes: leaves at l_c with n_points > n_s;
  * phi_S = W * type1((y - c_S) h/sqrt(delta), q, eps/10, sign=-1);
  * target-centric lists: L_P(T) = dense neighbours (incl. self) with image shift v,
    L_D(T) = all other touching leaves with sources;
  * psi_T = sum exp(i k.(c_T - c_S - v)) phi_S;  u += Re type2((x - c_T) sc, psi, +1);
  * direct: gauss_sum(x_T, y_S + v, q_S, 1/delta, r2_cut = D0^2 delta).
"""

import time

import numpy as np

from . import kernels, nufft
from .params import clamp_eps, periodic_kernel_1d, quad
from .tree import build, offsets


def neighbour_lists(tree, T):
    """Neighbour leaves of leaf T as [(S, v)], deduplicated on (S, v)."""
    l = tree.level[T]
    g = tree.coords[T]
    side = 2 ** l
    if not hasattr(tree, "_maps"):
        tree._maps = {}
        for b in range(tree.n_boxes):
            tree._maps[(int(tree.level[b]),) + tuple(int(c) for c in tree.coords[b])] = b

    def covering(lv, cell):
        c = np.asarray(cell)
        for ll in range(lv, -1, -1):
            b = tree._maps.get((ll,) + tuple(int(x) for x in c))
            if b is not None:
                return b
            c = c >> 1
        raise RuntimeError("no covering box")

    seen, out = set(), []
    for o in offsets(tree.dim):
        n = g + o
        if tree.periodic:
            v = n // side
            n = n - v * side
        else:
            if np.any(n < 0) or np.any(n >= side):
                continue
            v = np.zeros(tree.dim, dtype=np.int64)
        nb = covering(l, n)
        cands = [nb]
        if not tree.is_leaf[nb]:
            cands = []
            for ch in tree.children[nb]:
                gc = tree.coords[ch] + 2 * v * side
                if np.all(gc >= 2 * g - 1) and np.all(gc <= 2 * g + 2):
                    cands.append(ch)
        for S in cands:
            key = (int(S),) + tuple(int(x) for x in v)
            if key not in seen:
                seen.add(key)
                out.append((int(S), v.copy()))
    return out


class Alg2:
    """The five phases of Alg 2 on one problem; each phase can be timed separately."""

    def __init__(self, sources, charges, targets, delta, epsilon, n_s, boundary="free"):
        self.periodic = boundary == "periodic"
        self.src = np.atleast_2d(np.asarray(sources, dtype=float))
        self.tgt = np.atleast_2d(np.asarray(targets, dtype=float))
        self.q = np.asarray(charges, dtype=float)
        self.delta, self.n_s = float(delta), int(n_s)
        self.eps = clamp_eps(epsilon)
        self.dim = self.src.shape[1]

    def build_tree(self):
        t = build(self.src, self.tgt, self.n_s, self.delta, self.eps, periodic=self.periodic)
        self.tree = t
        self.pw = quad(self.eps, self.delta, R=t.R, dim=self.dim)
        self.sc = self.pw.h / np.sqrt(self.delta)
        self.W = self.pw.wtensor()
        self.ctr = t.centers()
        self.dense = np.nonzero(t.is_leaf & (t.level == t.l_c) & (t.n_points > self.n_s))[0]
        self.is_dense = np.zeros(t.n_boxes, dtype=bool)
        self.is_dense[self.dense] = True
        self.tleaves = np.nonzero(t.is_leaf & (t.tgt_count > 0))[0]
        self.u_sorted = np.zeros(self.tgt.shape[0])
        self.tgt_sorted = self.tgt[t.tgt_perm]
        self.lists = {}
        return t

    def _src(self, b):
        t = self.tree
        idx = t.src_perm[t.src_start[b]:t.src_start[b] + t.src_count[b]]
        return self.src[idx], self.q[idx]

    def _tgt_slice(self, b):
        t = self.tree
        return slice(t.tgt_start[b], t.tgt_start[b] + t.tgt_count[b])

    def list_of(self, T):
        if T not in self.lists:
            self.lists[T] = neighbour_lists(self.tree, T)
        return self.lists[T]

    def form(self, boxes=None):
        """Outgoing expansions of the P-boxes (Alg 2 step 1)."""
        self.phi = getattr(self, "phi", {})
        for S in (self.dense if boxes is None else boxes):
            y, q = self._src(S)
            f = nufft.type1((y - self.ctr[S]) * self.sc, q.astype(np.complex128), self.pw.n_f,
                            self.dim, self.eps / 10, sign=-1)
            self.phi[S] = self.W * f

    def _phase(self, delta_vec):
        k = self.pw.m * self.sc
        p = np.exp(1j * k * delta_vec[0])
        for ax in range(1, self.dim):
            p = np.multiply.outer(p, np.exp(1j * k * delta_vec[ax]))
        return p

    def gather_eval(self, targets=None):
        """Translate (gather) then evaluate incoming expansions (Alg 2 steps 2-3)."""
        t = self.tree
        tgt_sorted = self.tgt_sorted
        for T in (self.tleaves if targets is None else targets):
            if t.level[T] != t.l_c:
                continue
            plist = [(S, v) for S, v in self.list_of(T) if self.is_dense[S]]
            if not plist:
                continue
            psi = np.zeros((self.pw.n_f,) * self.dim, dtype=np.complex128)
            for S, v in plist:
                psi += self._phase(self.ctr[T] - self.ctr[S] - v * t.root_side) * self.phi[S]
            sl = self._tgt_slice(T)
            x = (tgt_sorted[sl] - self.ctr[T]) * self.sc
            val = nufft.type2(x, psi, self.pw.n_f, self.dim, self.eps / 10, sign=+1)
            self.u_sorted[sl] += val.real

    def direct(self, targets=None):
        """Direct interactions over the D-lists with the ball cut (Alg 2 step 4)."""
        t = self.tree
        tgt_sorted = self.tgt_sorted
        r2 = self.pw.D0 ** 2 * self.delta
        for T in (self.tleaves if targets is None else targets):
            sl = self._tgt_slice(T)
            for S, v in self.list_of(T):
                if self.is_dense[S] or t.src_count[S] == 0:
                    continue
                y, q = self._src(S)
                kernels.gauss_sum(tgt_sorted[sl], y + v * t.root_side, q, 1.0 / self.delta, r2,
                                  self.u_sorted[sl])

    def potentials(self):
        u = np.empty_like(self.u_sorted)
        u[self.tree.tgt_perm] = self.u_sorted
        return u


def fgt_points(sources, charges, targets, delta, epsilon, n_s, boundary="free", timings=None):
    """Oracle Alg 2: potentials at the targets (optionally per-phase wall times)."""
    a = Alg2(sources, charges, targets, delta, epsilon, n_s, boundary)
    t0 = time.perf_counter()
    a.build_tree()
    t1 = time.perf_counter()
    a.form()
    t2 = time.perf_counter()
    a.gather_eval()
    t3 = time.perf_counter()
    a.direct()
    t4 = time.perf_counter()
    if timings is not None:
        timings.update(tree=t1 - t0, form=t2 - t1, gather_eval=t3 - t2, direct=t4 - t3)
    return a.potentials()


def fgt_points_periodic_root(sources, charges, targets, delta, epsilon):
    """Periodic transform in the root Fourier-series regime (cutoff level <= 1):
    PAPER.md:1449-1453 ("the plane-wave expansion of the periodic Gaussian G_p on the
    entire box B ... can be used directly"), series PAPER.md:363-383 with n_p
    and coefficients of planewave.periodic_params (planewave.py:148-155):

        u_i = Re sum_{n in [-n_p, n_p]^d} prod_k c(n_k) e^{2 pi i n.x_i} sum_j q_j e^{-2 pi i n.y_j}

    computed as dense separable DFTs (small problems only)."""
    src = np.atleast_2d(np.asarray(sources, dtype=float))
    tgt = np.atleast_2d(np.asarray(targets, dtype=float))
    q = np.asarray(charges, dtype=float)
    d = tgt.shape[1] if tgt.size else src.shape[1]
    eps = clamp_eps(epsilon)
    n_p = int(np.ceil(np.sqrt(np.log(1.0 / eps)) / (np.pi * np.sqrt(delta))))
    n = np.arange(-n_p, n_p + 1)
    c = np.sqrt(np.pi * delta) * np.exp(-(np.pi * np.sqrt(delta) * n) ** 2)
    # outgoing: phi[n_0, .., n_{d-1}] = prod_k c(n_k) sum_j q_j prod_k e^{-2 pi i n_k y_jk}
    E = [np.exp(-2j * np.pi * np.multiply.outer(src[:, k], n)) for k in range(d)]
    if d == 1:
        phi = q @ E[0]
    elif d == 2:
        phi = np.einsum("j,ja,jb->ab", q, E[0], E[1])
    else:
        phi = np.einsum("j,ja,jb,jc->abc", q, E[0], E[1], E[2])
    for k in range(d):
        shape = [1] * d
        shape[k] = -1
        phi = phi * c.reshape(shape)
    # evaluation at the targets
    F = [np.exp(2j * np.pi * np.multiply.outer(tgt[:, k], n)) for k in range(d)]
    if d == 1:
        u = F[0] @ phi
    elif d == 2:
        u = np.einsum("ia,ib,ab->i", F[0], F[1], phi)
    else:
        u = np.einsum("ia,ib,ic,abc->i", F[0], F[1], F[2], phi)
    return u.real


def direct_oracle(sources, charges, targets, delta, boundary="free"):
    """Exact O(NM) sums; periodic via per-axis periodic kernels."""
    src = np.atleast_2d(np.asarray(sources, dtype=float))
    tgt = np.atleast_2d(np.asarray(targets, dtype=float))
    q = np.asarray(charges, dtype=float)
    out = np.zeros(tgt.shape[0])
    if boundary == "free":
        return kernels.gauss_sum(tgt, src, q, 1.0 / delta, np.inf, out)
    for a in range(0, tgt.shape[0], 256):
        diff = tgt[a:a + 256, None, :] - src[None, :, :]
        g = np.prod(periodic_kernel_1d(diff, delta), axis=-1)
        out[a:a + 256] = g @ q
    return out
