"""GPU parity of the continuous (box) FGT: libfgtcuda.so vs the CPU oracle and vs closed
forms (SPEC.md:651 acceptance 7)."""

import numpy as np
import pytest

from oracle import volume as ov

pytestmark = pytest.mark.gpu


def gaussians(d):
    C = np.array([[0.1, -0.05, 0.02][:d], [-0.2, 0.15, -0.1][:d]])
    W, A = [0.05, 0.1], [1.0, 0.7]
    return (lambda p: sum(a * np.exp(-np.sum((p - c) ** 2, axis=-1) / w ** 2)
                          for c, w, a in zip(C, W, A))), C, W, A


def rel_err(u, ref):
    num = sum(np.sum((u[b] - ref[b]) ** 2) for b in ref)
    den = sum(np.sum(ref[b] ** 2) for b in ref)
    return np.sqrt(num / den)


CASES = [  # d, k, delta, eps
    (1, 12, 1e-3, 1e-9),
    (2, 10, 1e-3, 1e-8),
    (2, 16, 1e-4, 1e-10),
    (3, 6, 1e-2, 1e-6),
    (3, 8, 1e-3, 1e-7),
]


@pytest.mark.parametrize("case", CASES, ids=[f"d{c[0]}k{c[1]}" for c in CASES])
def test_box_fgt_vs_oracle_and_closed_form(cuda, case):
    from paper_2305_07165_b200 import volume as pv
    d, k, delta, eps = case
    dens, C, W, A = gaussians(d)
    tree, vals, _ = pv.build_density_tree(dens, d, k, eps * 0.1)
    u = pv.fgt_box(tree, vals, delta, eps)
    to = ov.density_tree(dens, d, k, eps * 0.1)
    assert np.array_equal(to.level, tree.level) and np.array_equal(to.coords, tree.coords)
    ref = ov.fgt_box(to, delta, eps)
    assert set(u) == set(ref)
    assert rel_err(u, ref) < 1e-11
    exact = {b: ov.gaussian_box_convolution(to.leaf_points(b), delta, C, W, A) for b in ref}
    assert rel_err(u, exact) <= 10 * eps


def test_box_fgt_constant_density(cuda):
    from scipy.special import erf
    from paper_2305_07165_b200 import volume as pv
    tree, vals, _ = pv.build_density_tree(lambda p: np.ones(p.shape[:-1]), 3, 6, 1e-10)
    delta, eps = 1e-2, 1e-8
    u = pv.fgt_box(tree, vals, delta, eps)
    for b, ub in u.items():
        x = pv.leaf_grid(tree, b, pv.LegendreBasis(6))
        ex = np.prod(np.sqrt(np.pi * delta) / 2 * (erf((0.5 - x) / np.sqrt(delta))
                                                   + erf((0.5 + x) / np.sqrt(delta))), axis=-1)
        assert np.max(np.abs(ub - ex)) <= 10 * eps * np.max(ex)


@pytest.mark.parametrize("d", [2, 3])
def test_box_fgt_periodic_eigenfunction(cuda, d):
    """sigma_p -> (pi delta)^{d/2} exp(-d pi^2 delta n^2) sigma_p."""
    from paper_2305_07165_b200 import volume as pv
    # 3-D kept small: phi/psi are stored for every f=1 box (n_f^3 modes each)
    n, delta, eps = (4, 1e-3, 1e-8) if d == 2 else (2, 2e-3, 1e-6)

    def sig(p):
        out = np.sin(2 * np.pi * n * p[..., 0])
        for ax in range(1, d):
            out = out * np.cos(2 * np.pi * n * p[..., ax])
        return out
    tree, vals, _ = pv.build_density_tree(sig, d, 8 if d == 2 else 6, 1e-9 if d == 2 else 1e-7,
                                           periodic=True)
    u = pv.fgt_box(tree, vals, delta, eps, boundary="periodic")
    fac = (np.pi * delta) ** (d / 2) * np.exp(-d * np.pi ** 2 * delta * n * n)
    num = den = 0.0
    for b, ub in u.items():
        ex = fac * sig(pv.leaf_grid(tree, b, pv.LegendreBasis(8 if d == 2 else 6)))
        num += np.sum((ub - ex) ** 2)
        den += np.sum(ex ** 2)
    assert np.sqrt(num / den) <= 10 * eps


def test_box_fgt_device_path(cuda):
    import torch
    from paper_2305_07165_b200 import volume as pv
    dens = gaussians(3)[0]
    tree, vals, _ = pv.build_density_tree(dens, 3, 8, 1e-8)
    plan = pv.BoxPlan(tree, 1e-3, 1e-7, 8, False)
    u = pv.fgt_box(tree, vals, 1e-3, 1e-7, plan=plan)
    leaves, V = pv._stack_values(tree, vals, 8)
    ud = pv.fgt_box_device(plan, torch.from_numpy(V).cuda())
    torch.cuda.synchronize()
    ud = ud.cpu().numpy()
    assert all(np.array_equal(ud[i], u[int(b)]) for i, b in enumerate(leaves))


@pytest.mark.parametrize("d,delta,eps,n", [(1, 0.05, 1e-10, 3), (2, 0.03, 1e-9, 2), (2, 0.02, 1e-12, 1),
                                           (3, 0.1, 1e-7, 1)])
def test_box_fgt_periodic_root_series(cuda, d, delta, eps, n):
    """Root Fourier-series regime (cutoff level <= 1): eigenfunctions
    sigma_n -> (pi delta)^{d/2} exp(-d pi^2 delta n^2) sigma_n, and a constant density on a
    single-leaf tree -> (pi delta)^{d/2} sigma."""
    from paper_2305_07165_b200 import volume as pv
    k = 10 if d < 3 else 8

    def sig(p):
        out = np.sin(2 * np.pi * n * p[..., 0])
        for ax in range(1, d):
            out = out * np.cos(2 * np.pi * n * p[..., ax])
        return out
    tree, vals, _ = pv.build_density_tree(sig, d, k, 1e-11 if d < 3 else 1e-8, periodic=True)
    plan = pv.BoxPlan(tree, delta, eps, k, True)
    assert plan.root_series and plan.l_c == 0 and plan.d_tgt.size == 0
    u = pv.fgt_box(tree, vals, delta, eps, boundary="periodic", plan=plan)
    fac = (np.pi * delta) ** (d / 2) * np.exp(-d * np.pi ** 2 * delta * n * n)
    num = den = 0.0
    for b, ub in u.items():
        ex = fac * sig(pv.leaf_grid(tree, b, pv.LegendreBasis(k)))
        num += np.sum((ub - ex) ** 2)
        den += np.sum(ex ** 2)
    assert np.sqrt(num / den) <= 10 * eps
    # constant density: the root stays a single leaf
    tree, vals, _ = pv.build_density_tree(lambda p: np.full(p.shape[:-1], 2.5), d, k, 1e-12, periodic=True)
    assert tree.n_boxes == 1
    u = pv.fgt_box(tree, vals, delta, eps, boundary="periodic")
    ex = 2.5 * (np.pi * delta) ** (d / 2)
    for ub in u.values():
        assert np.max(np.abs(ub - ex)) <= 10 * eps * ex


def _vol_cases(n=8, seed=7):
    r = np.random.default_rng(seed)
    out = []
    for i in range(n):
        d = int(r.integers(1, 4))
        k = int(r.integers(4, 13 if d < 3 else 9))
        delta = float(10.0 ** r.uniform(-3.5, -1.5))
        eps = float(10.0 ** -r.integers(4, 11 if d < 3 else 8))
        out.append((f"v{i}", d, k, delta, eps, int(r.integers(1, 4))))
    return out


VSWEEP = _vol_cases()


@pytest.mark.parametrize("case", VSWEEP, ids=[c[0] for c in VSWEEP])
def test_box_fgt_random_sweep(cuda, case):
    """Seeded random (d, k, delta, eps, Gaussian mixture): density tree bit-exact vs the
    oracle, GPU transform vs the oracle Alg 4 (<= 1e-10 relative) and vs the closed-form
    Gaussian convolution (<= 10 eps)."""
    from paper_2305_07165_b200 import volume as pv
    name, d, k, delta, eps, ng = case
    r = np.random.default_rng(int(name[1:]) + 31)
    C = r.uniform(-0.3, 0.3, (ng, d))
    W = r.uniform(0.03, 0.15, ng)
    A = r.uniform(0.5, 1.5, ng)
    dens = lambda p: sum(a * np.exp(-np.sum((p - c) ** 2, axis=-1) / w ** 2)  # noqa: E731
                         for c, w, a in zip(C, W, A))
    tree, vals, _ = pv.build_density_tree(dens, d, k, max(eps * 0.1, 1e-12))
    to = ov.density_tree(dens, d, k, max(eps * 0.1, 1e-12))
    assert np.array_equal(to.level, tree.level) and np.array_equal(to.coords, tree.coords)
    u = pv.fgt_box(tree, vals, delta, eps)
    ref = ov.fgt_box(to, delta, eps)
    assert rel_err(u, ref) < 1e-10
    exact = {b: ov.gaussian_box_convolution(to.leaf_points(b), delta, C, W, A) for b in ref}
    assert rel_err(u, exact) <= 10 * eps


@pytest.mark.parametrize("d", [1, 2, 3])
def test_interp_at(cuda, d):
    """interp_at: exact for polynomials of degree < k, the stored value
    at a grid node, and the transform's closed form at random points."""
    from paper_2305_07165_b200 import volume as pv
    k = 8
    dens, C, W, A = gaussians(d)
    tree, vals, _ = pv.build_density_tree(dens, d, k, 1e-9)
    leaves = np.nonzero(tree.is_leaf)[0]
    basis = pv.LegendreBasis(k)
    r = np.random.default_rng(40 + d)
    # (1) a polynomial of degree k-1 per axis is reproduced to roundoff
    poly = lambda p: np.prod(1.0 + 0.3 * p + 0.2 * p ** 3 - 0.1 * p ** (k - 1), axis=-1)  # noqa: E731
    pots = {int(b): poly(pv.leaf_grid(tree, b, basis)) for b in leaves}
    x = r.uniform(-0.5, 0.5, (5000, d))
    assert np.max(np.abs(pv.interp_at(tree, pots, x) - poly(x))) < 1e-12
    # (2) grid nodes of a leaf give the stored values
    b = int(leaves[len(leaves) // 2])
    g = pv.leaf_grid(tree, b, basis).reshape(-1, d)
    assert np.max(np.abs(pv.interp_at(tree, pots, g) - pots[b].reshape(-1))) < 1e-12
    # (3) the transform at random points vs the closed-form Gaussian convolution
    delta, eps = 1e-3, 1e-9
    u = pv.fgt_box(tree, vals, delta, eps)
    ui = pv.interp_at(tree, u, x)
    from oracle import volume as ov
    ex = ov.gaussian_box_convolution(x, delta, C, W, A)
    assert np.linalg.norm(ui - ex) / np.linalg.norm(ex) < 1e-7


def test_refine_output_alg5(cuda):
    """Alg 5: leaves whose potential fails the tail test are refined
    until every leaf passes (up to the input tree's depth, Alg 5 Remark); the refined
    potentials agree with the old ones at the old grid nodes (value consistency) and the
    source density is unchanged (exact polynomial refill)."""
    from paper_2305_07165_b200 import volume as pv
    d, k, eps, delta, w = 2, 5, 1e-8, 5e-3, 0.12
    dens = lambda p: np.exp(-np.sum((p - 0.1) ** 2, axis=-1) / w ** 2)  # noqa: E731
    tree, vals, _ = pv.build_density_tree(dens, d, k, 1e-5)
    u = pv.fgt_box(tree, vals, delta, eps)
    basis = pv.LegendreBasis(k)
    tail = lambda v: pv.tail_error(pv.apply_per_axis(basis.val_to_pol, np.asarray(v).reshape((k,) * d), d))  # noqa: E731
    lmax = int(tree.level.max())
    assert any(tail(v) > eps and tree.level[b] < lmax for b, v in u.items())
    t2, v2, u2, rounds = pv.refine_output(tree, vals, u, delta, eps)
    assert rounds >= 1 and t2.n_boxes > tree.n_boxes and int(t2.level.max()) <= lmax
    assert all(tail(v) <= eps for b, v in u2.items() if t2.level[b] < lmax)
    nodes = np.concatenate([pv.leaf_grid(tree, b, basis).reshape(-1, d) for b in u])
    old = np.concatenate([np.asarray(u[b]).reshape(-1) for b in u])
    # (the tail test is an absolute error estimate, Eq. funerr)
    assert np.max(np.abs(pv.interp_at(t2, u2, nodes) - old)) <= 10 * eps
    x = np.random.default_rng(51).uniform(-0.5, 0.5, (3000, d))
    assert np.max(np.abs(pv.interp_at(t2, v2, x) - pv.interp_at(tree, vals, x))) < 1e-12
