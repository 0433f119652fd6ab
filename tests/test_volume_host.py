"""CPU tests of the volume FGT host side (no GPU): Alg 3 tree vs the reference fixtures,
the 1-D tables vs the oracle, and the plan's lists / flags vs the oracle's."""

import os

import numpy as np
import pytest

from oracle import volume as ov

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sigma_f(d):
    C = np.array([[0.1, -0.05, 0.02][:d], [-0.2, 0.15, -0.1][:d]])
    W, A = [0.05, 0.1], [1.0, 0.7]
    return lambda p: sum(a * np.exp(-np.sum((p - c) ** 2, axis=-1) / w ** 2) for c, w, a in zip(C, W, A))


@pytest.mark.parametrize("d,k,eps", [(2, 10, 1e-9), (3, 6, 1e-7)])
def test_product_density_tree_vs_reference(d, k, eps):
    from paper_2305_07165_b200 import volume as pv
    g = np.load(os.path.join(GOLD, f"dtree_{d}d.npz"))
    t, vals, coeffs = pv.build_density_tree(sigma_f(d), d, k, eps)
    for f in ("level", "parent", "children", "coords", "is_leaf"):
        assert np.array_equal(getattr(t, f), g[f]), f
    V = np.stack([vals[b] for b in g["leaves"]]).reshape(len(g["leaves"]), -1)
    assert np.allclose(V.sum(axis=1), g["vsum"], rtol=1e-13, atol=1e-13)
    b0 = int(g["leaves"][0])
    assert np.allclose(pv.apply_per_axis(pv.LegendreBasis(k).pol_to_val, coeffs[b0], d), vals[b0])


def test_refill_interpolate_rejected():
    from paper_2305_07165_b200 import volume as pv
    with pytest.raises(ValueError):
        pv.build_density_tree(sigma_f(2), 2, 6, 1e-6, refill="interpolate")


def test_moment_tables_match_oracle():
    from paper_2305_07165_b200 import volume as pv
    t = np.linspace(-3, 3, 61)
    for lam in (1 / 64, 0.1, 0.64, 2.0):
        a, b = pv.gauss_moment_J(lam, 15, t), ov.gauss_J(lam, 15, t)
        assert np.max(np.abs(a - b)) < 1e-12 * lam
    tt = np.linspace(-60, 60, 121)
    assert np.max(np.abs(pv.fourier_moment_I(20, tt) - ov.fourier_I(20, tt))) < 1e-15


@pytest.mark.parametrize("periodic", [False, True])
def test_box_plan_lists_match_oracle(periodic):
    from paper_2305_07165_b200 import volume as pv
    d, k, delta, eps = 2, 8, 1e-4, 1e-8
    # constant-plus-bump density: leaves at coarse levels give direct pairs as well
    dens = lambda p: 0.3 + sigma_f(d)(p)  # noqa: E731
    t, vals, _ = pv.build_density_tree(dens, d, k, 1e-9, periodic=periodic)
    plan = pv.BoxPlan(t, delta, eps, k, periodic)
    to = ov.density_tree(dens, d, k, 1e-9, periodic=periodic)
    f, pw_pairs, d_pairs = ov.box_lists(to, plan.l_c)
    assert plan.n_pw == int(f.sum())
    assert plan.n_gather_pairs == len(pw_pairs)
    leaves = np.nonzero(to.is_leaf)[0]
    slot = {int(b): i for i, b in enumerate(leaves)}
    want = sorted((slot[T], slot[S]) for T, S, _ in d_pairs)
    got = sorted(zip(plan.d_tgt.tolist(), plan.d_src.tolist()))
    assert got == want
    # every direct pair references 11-offset tables of the source level only
    assert plan.d_tab.size > 0 and plan.d_tab.max() < plan.dtab.shape[0]


def test_coarsen_output_alg6():
    """Alg 6: an over-refined smooth potential collapses toward the root
    and the kept leaves still hold the function to ~epsilon; a constant collapses fully."""
    from paper_2305_07165_b200 import volume as pv
    d, k = 2, 8
    tree, vals, _ = pv.build_density_tree(lambda p: np.exp(-np.sum(p ** 2, axis=-1) / 0.01), d, k, 1e-10)
    basis = pv.LegendreBasis(k)
    f = lambda p: np.prod(np.cos(2 * p), axis=-1)  # noqa: E731
    pots = {int(b): f(pv.leaf_grid(tree, b, basis)) for b in np.nonzero(tree.is_leaf)[0]}
    t2, p2 = pv.coarsen_output(tree, pots, 1e-9)
    assert t2.n_boxes < tree.n_boxes and set(p2) == set(np.nonzero(t2.is_leaf)[0].tolist())
    assert max(np.max(np.abs(v - f(pv.leaf_grid(t2, b, basis)))) for b, v in p2.items()) < 1e-8
    # renumbered tree is consistent: parents/children point at live boxes of the right level
    for b in range(t2.n_boxes):
        if t2.parent[b] >= 0:
            assert t2.level[t2.parent[b]] == t2.level[b] - 1
        for c in t2.children[b]:
            assert (c < 0) == bool(t2.is_leaf[b])
    const = {int(b): np.full((k,) * d, 3.0) for b in np.nonzero(tree.is_leaf)[0]}
    t3, p3 = pv.coarsen_output(tree, const, 1e-12)
    assert t3.n_boxes == 1 and np.allclose(p3[0], 3.0)


@pytest.mark.parametrize("d,periodic", [(2, True), (2, False), (3, False)])
def test_direct_table_key_matches_plan_offsets(d, periodic):
    """The integer-coordinate key Alg 5 uses for its extended T_pol2pot tables
    (direct_table_key) reproduces, on every leaf pair of the plan's D-lists, the (offset,
    ratio) the Alg 4 plan reads from box centres -- one of the 11 standard offsets -- so the
    standard tables are the level-restricted special case of the extended ones."""
    from paper_2305_07165_b200 import volume as pv
    k, delta, eps = 6, 1e-4, 1e-8
    dens = lambda p: 0.3 + sigma_f(d)(p)  # noqa: E731
    t, vals, _ = pv.build_density_tree(dens, d, k, 1e-4 if d == 2 else 1e-2, periodic=periodic)
    plan = pv.BoxPlan(t, delta, eps, k, periodic)
    assert plan.d_sources
    ctr = t.centers()
    n = 0
    for T, lst in plan.d_sources.items():
        for S_slot, ls, gs, v in lst:
            S = int(plan.leaves[S_slot])
            offs, r = pv.direct_table_key(int(t.level[T]), t.coords[T], ls, gs, v)
            Ls = t.root_side / 2.0 ** ls
            want = (ctr[T] - ctr[S] - np.asarray(v) * t.root_side) / Ls
            assert np.allclose(offs, want, rtol=0, atol=1e-12) and r == 2.0 ** (ls - int(t.level[T]))
            assert all((o, r) in pv.OFFSETS for o in offs)
            n += 1
    assert n == plan.d_tgt.size
    if periodic:
        assert any(any(v) for lst in plan.d_sources.values() for _, _, _, v in lst)
