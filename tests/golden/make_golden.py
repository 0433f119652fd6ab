"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports /root/reference/pkg/src/fgt read-only and writes compressed .npz fixtures
next to this file.  Nothing at test time reads /root/reference; the fixtures travel.

Fixtures:
  params.npz    Table 1 n_f / h / D0 for R in {2,3,4} D0 (planewave.pw_params),
                Table 2 n_p (planewave.periodic_params), cutoff_level cases (tree.py)
  kernels.npz   _kernels_py.gauss_direct(_periodic), nufft_spread / nufft_interp
  nufft.npz     nufft.nufft_type1 / nufft_type2 (direct and grid paths), dft_oracle
  tree_*.npz    tree.build_point_tree outputs (Tree + PointPartition, creation-order ids)
  alg2_cfg1.npz Alg 2 potentials composed from the reference primitives (tree,
                nufft_type1/2, gauss_direct) for BASELINE config 1, plus the exact
                O(NM) sums (gauss_direct with r2_cut = inf)
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import fgt.backend as rb  # noqa: E402
from fgt import nufft as rn  # noqa: E402
from fgt import planewave as rp  # noqa: E402
from fgt import tree as rt  # noqa: E402

assert rb.BACKEND == "python"


def save(name, **arrs):
    np.savez_compressed(os.path.join(HERE, name), **arrs)
    print("wrote", name, {k: getattr(v, "shape", None) for k, v in arrs.items()})


def params():
    eps = np.array([1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8, 1e-9, 1e-10, 1e-11, 1e-12])
    nf, h, D0 = np.zeros((3, eps.size), int), np.zeros((3, eps.size)), np.zeros(eps.size)
    for i, e in enumerate(eps):
        d0 = rp.cutoff_factor(e)
        D0[i] = d0
        for k, f in enumerate((2.0, 3.0, 4.0)):
            q = rp.pw_params(e, 1e-3, R=f * d0, dim=2)
            nf[k, i], h[k, i] = q.n_f, q.h
    w30 = rp.pw_params(1e-6, 1e-3, dim=3).weights_1d
    np_eps = np.array([1e-2, 1e-6, 1e-12])
    np_delta = np.array([1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6])
    n_p = np.array([[rp.periodic_params(e, dl).n_p for dl in np_delta] for e in np_eps])
    cl_cases = np.array([[1e-2, 1e-6, 1.0, 0], [1e-6, 1e-6, 1.0, 0], [1e-4, 1e-10, 1.0, 0],
                         [1e-5, 1e-8, 1.0, 0], [1e-3, 1e-6, 0.9934, 1], [1e-4, 1e-9, 0.98, 1],
                         [1e-6, 1e-6, 0.7, 1], [1.0, 1e-6, 0.5, 1]])
    cl_out = np.array([list(rt.cutoff_level(c[0], c[1], c[2], "point" if c[3] else "density"))
                       for c in cl_cases])
    save("params.npz", eps=eps, nf=nf, h=h, D0=D0, w30=w30, np_eps=np_eps, np_delta=np_delta,
         n_p=n_p, cl_cases=cl_cases, cl_out=cl_out)


def kernels():
    r = np.random.default_rng(100)
    out = {}
    for d in (1, 2, 3):
        t = r.uniform(-0.5, 0.5, (64, d))
        s = r.uniform(-0.5, 0.5, (97, d))
        q = r.standard_normal(97)
        out[f"gd_t{d}"], out[f"gd_s{d}"], out[f"gd_q{d}"] = t, s, q
        out[f"gd_free{d}"] = rb.gauss_direct(t, s, q, 50.0, 0.05, np.zeros(64))
        out[f"gd_inf{d}"] = rb.gauss_direct(t, s, q, 50.0, np.inf, np.zeros(64))
        out[f"gd_per{d}"] = rb.gauss_direct_periodic(t, s, q, 50.0, np.inf, np.zeros(64))
        n_r, m = (48, 6) if d < 3 else (20, 4)
        x = r.uniform(0, 2 * np.pi, (40, d))
        v = r.standard_normal(40) + 1j * r.standard_normal(40)
        g = np.zeros((n_r,) * d, complex)
        rb.nufft_spread(x, v, n_r, m, 0.02, g)
        grid = r.standard_normal((n_r,) * d) + 1j * r.standard_normal((n_r,) * d)
        out[f"sp_x{d}"], out[f"sp_v{d}"], out[f"sp_g{d}"] = x, v, g
        out[f"ip_grid{d}"] = grid
        out[f"ip_out{d}"] = rb.nufft_interp(x, grid, n_r, m, 0.02)
    save("kernels.npz", **out)


def nufft():
    r = np.random.default_rng(200)
    out = {}
    for d, n_f in ((1, 30), (2, 20), (3, 12)):
        grid = rn.ModeGrid(d, n_f)
        x = r.uniform(-np.pi, np.pi, (150, d))
        f = r.standard_normal(150) + 1j * r.standard_normal(150)
        c = r.standard_normal(grid.shape) + 1j * r.standard_normal(grid.shape)
        out[f"x{d}"], out[f"f{d}"], out[f"c{d}"] = x, f, c
        for eps in (1e-4, 1e-8, 1e-12):
            tag = f"{d}_{int(-np.log10(eps))}"
            out[f"t1grid_{tag}"] = rn.nufft_type1(x, f, grid, eps, sign=-1, method="grid")
            out[f"t2grid_{tag}"] = rn.nufft_type2(x, c, grid, eps, sign=+1, method="grid")
        out[f"t1dft_{d}"] = rn.dft_oracle(x, f, grid, "type1", -1)
        out[f"t2dft_{d}"] = rn.dft_oracle(x, c, grid, "type2", +1)
        out[f"plan_{d}"] = np.array(rn._plan(grid, 1e-10))
    save("nufft.npz", **out)


TREE_CASES = {
    # name: (generator, n_s, delta, eps, periodic)
    "cfg1": ("uniform2", 100, 1e-3, 1e-6, False),
    "clust3d": ("clust3", 40, 1e-4, 1e-9, False),
    "periodic2d": ("uniform2p", 50, 1e-4, 1e-8, True),
    "shell3d": ("shell3", 10, 1e-5, 1e-6, False),
}


def tree_inputs(gen):
    if gen == "uniform2":
        r = np.random.default_rng(0)
        y = r.uniform(-0.5, 0.5, (20000, 2))
        return y, y.copy(), r.uniform(-1, 1, 20000)
    if gen == "uniform2p":
        y = np.random.default_rng(0).uniform(-0.5, 0.5, (20000, 2))
        x = np.random.default_rng(1).uniform(-0.5, 0.5, (20000, 2))
        return y, x, None
    if gen == "clust3":
        r = np.random.default_rng(1)
        C = r.uniform(-0.5, 0.5, (8, 3))
        lab = r.integers(0, 8, 20000)
        y = np.clip(C[lab] + 0.02 * r.standard_normal((20000, 3)), -0.5, 0.5)
        x = np.random.default_rng(2).uniform(-0.5, 0.5, (20000, 3))
        return y, x, None
    r = np.random.default_rng(0)
    u = r.standard_normal((20000, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    y = (0.35 + 1e-3 * (r.uniform(size=20000) - 0.5))[:, None] * u
    x = np.random.default_rng(1).uniform(-0.5, 0.5, (20000, 3))
    return y, x, None


def trees():
    for name, (gen, n_s, delta, eps, periodic) in TREE_CASES.items():
        y, x, _ = tree_inputs(gen)
        t, p, l_c, R = rt.build_point_tree(y, x, n_s, delta, eps, periodic=periodic)
        save(f"tree_{name}.npz", level=t.level, parent=t.parent, children=t.children,
             coords=t.coords, is_leaf=t.is_leaf, root_center=t.root_center,
             root_side=np.array(t.root_side), src_perm=p.src_perm.astype(np.int32),
             tgt_perm=p.tgt_perm.astype(np.int32), src_start=p.src_start,
             src_count=p.src_count, tgt_start=p.tgt_start, tgt_count=p.tgt_count,
             n_points=p.n_points, l_c=np.array(l_c), R=np.array(R))


def alg2_cfg1():
    """Alg 2 composed from reference primitives (SURVEY §3B semantics), config 1."""
    y, x, q = tree_inputs("uniform2")
    delta, eps, n_s = 1e-3, 1e-6, 100
    t, p, l_c, R = rt.build_point_tree(y, x, n_s, delta, eps)
    pw = rp.pw_params(rp.clamp_tolerance(eps), delta, R=R, dim=2)
    grid = rn.ModeGrid(2, pw.n_f)
    sc = pw.h / np.sqrt(delta)
    W = pw.weights_tensor()
    ctr = t.centers()
    dense = t.is_leaf & (t.level == l_c) & (p.n_points > n_s)
    phi = {}
    for S in np.nonzero(dense)[0]:
        idx = p.src_perm[p.src_start[S]:p.src_start[S] + p.src_count[S]]
        phi[S] = W * rn.nufft_type1((y[idx] - ctr[S]) * sc, q[idx], grid, eps / 10, sign=-1)
    k = pw.modes * sc
    u = np.zeros(x.shape[0])
    r2 = pw.D0 ** 2 * delta
    for T in np.nonzero(t.is_leaf & (p.tgt_count > 0))[0]:
        ti = p.tgt_perm[p.tgt_start[T]:p.tgt_start[T] + p.tgt_count[T]]
        lvl, g = t.level[T], t.coords[T]
        nbrs, seen = [], set()
        for o in rt._offsets(2):
            n = g + o
            if np.any(n < 0) or np.any(n >= 2 ** lvl):
                continue
            b = t.find_covering(lvl, n)
            cands = [b] if t.is_leaf[b] else [
                c for c in t.children[b]
                if np.all(t.coords[c] >= 2 * g - 1) and np.all(t.coords[c] <= 2 * g + 2)]
            for c in cands:
                if c not in seen:
                    seen.add(c)
                    nbrs.append(c)
        psi = None
        for S in nbrs:
            if dense[S]:
                dv = ctr[T] - ctr[S]
                ph = np.multiply.outer(np.exp(1j * k * dv[0]), np.exp(1j * k * dv[1]))
                psi = ph * phi[S] if psi is None else psi + ph * phi[S]
            elif p.src_count[S] > 0:
                si = p.src_perm[p.src_start[S]:p.src_start[S] + p.src_count[S]]
                acc = np.zeros(ti.size)
                rb.gauss_direct(x[ti], y[si], q[si], 1.0 / delta, r2, acc)
                u[ti] += acc
        if psi is not None:
            u[ti] += rn.nufft_type2((x[ti] - ctr[T]) * sc, psi, grid, eps / 10, sign=+1).real
    exact = rb.gauss_direct(x, y, q, 1.0 / delta, np.inf, np.zeros(x.shape[0]))
    save("alg2_cfg1.npz", u=u, exact=exact)


def sigma_f(d):
    """Sum of two Gaussians (the density used by the volume fixtures)."""
    C = np.array([[0.1, -0.05, 0.02][:d], [-0.2, 0.15, -0.1][:d]])
    W, A = [0.05, 0.1], [1.0, 0.7]
    return lambda p: sum(a * np.exp(-np.sum((p - c) ** 2, axis=-1) / w ** 2) for c, w, a in zip(C, W, A))


def volume():
    from fgt import poly1d as rpoly
    out = {}
    # Gaussian moments: recurrence window and quadrature window (poly1d.py:129-195)
    t = np.linspace(-3, 3, 61)
    for lam in (1 / 64, 1 / 32, 1 / 16, 1 / 8, 0.25, 0.64):
        out[f"J_{lam:.6f}"] = rpoly.gauss_moment_J(lam, 15, t)
    tI = np.linspace(-100, 100, 401)
    out["I"] = rpoly.fourier_moment_I(23, tI)
    b = rpoly.LegendreBasis.build(12)
    out["nodes12"], out["v2p12"], out["p2v12"] = b.nodes, b.val_to_pol, b.pol_to_val
    r = np.random.default_rng(3)
    c = r.standard_normal((6, 6, 6))
    out["tail_c"], out["tail"] = c, np.array(rpoly.tail_error(c))
    save("poly1d.npz", **out)
    for d, k, eps in ((2, 10, 1e-9), (3, 6, 1e-7)):
        t, vals, _ = rt.build_density_tree(sigma_f(d), d, k, eps)
        leaves = np.nonzero(t.is_leaf)[0]
        V = np.stack([vals[b] for b in leaves]).reshape(len(leaves), -1)
        save(f"dtree_{d}d.npz", level=t.level, parent=t.parent, children=t.children,
             coords=t.coords, is_leaf=t.is_leaf, leaves=leaves,
             vsum=V.sum(axis=1), vsq=(V * V).sum(axis=1))


if __name__ == "__main__":
    params()
    kernels()
    nufft()
    trees()
    alg2_cfg1()
    volume()
