"""Pin the CPU oracle against golden fixtures produced by the real reference package
(tests/golden/make_golden.py).  CPU only."""

import os

import numpy as np
import pytest

from oracle import kernels as ok
from oracle import nufft as on
from oracle import params as op
from oracle import point_fgt as ofgt
from oracle import tree as ot

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_table1_and_weights_exact():
    g = load("params.npz")
    for i, e in enumerate(g["eps"]):
        assert op.d0_of(e) == g["D0"][i]
        for k, f in enumerate((2.0, 3.0, 4.0)):
            q = op.quad(e, 1e-3, R=f * op.d0_of(e), dim=2)
            assert q.n_f == g["nf"][k, i] and q.h == g["h"][k, i]
    # the paper's Table 1
    assert list(g["nf"][0, [0, 2, 4, 6, 8, 10]]) == [12, 20, 30, 38, 48, 56]
    assert list(g["nf"][2, [0, 2, 4, 6, 8, 10]]) == [20, 34, 48, 64, 78, 92]
    assert np.array_equal(op.quad(1e-6, 1e-3, dim=3).w1, g["w30"])


def test_table2_and_cutoff_level_exact():
    g = load("params.npz")
    for i, e in enumerate(g["np_eps"]):
        for j, dl in enumerate(g["np_delta"]):
            assert op.periodic_np(e, dl) == g["n_p"][i, j]
    for c, out in zip(g["cl_cases"], g["cl_out"]):
        l_c, R = op.cut_level(c[0], c[1], c[2], "point" if c[3] else "density")
        assert l_c == out[0] and R == out[1]


@pytest.mark.parametrize("d", [1, 2, 3])
def test_kernels(d):
    g = load("kernels.npz")
    t, s, q = g[f"gd_t{d}"], g[f"gd_s{d}"], g[f"gd_q{d}"]
    assert rel(ok.gauss_sum(t, s, q, 50.0, 0.05, np.zeros(64)), g[f"gd_free{d}"]) < 1e-14
    assert rel(ok.gauss_sum(t, s, q, 50.0, np.inf, np.zeros(64)), g[f"gd_inf{d}"]) < 1e-14
    assert rel(ok.gauss_sum(t, s, q, 50.0, np.inf, np.zeros(64), periodic=True),
               g[f"gd_per{d}"]) < 1e-14
    n_r, m = (48, 6) if d < 3 else (20, 4)
    x, v = g[f"sp_x{d}"], g[f"sp_v{d}"]
    assert rel(ok.spread(x, v, n_r, m, 0.02, np.zeros((n_r,) * d, complex)), g[f"sp_g{d}"]) < 1e-14
    assert rel(ok.interp(x, g[f"ip_grid{d}"], n_r, m, 0.02), g[f"ip_out{d}"]) < 1e-14


@pytest.mark.parametrize("d,n_f", [(1, 30), (2, 20), (3, 12)])
def test_nufft(d, n_f):
    g = load("nufft.npz")
    x, f, c = g[f"x{d}"], g[f"f{d}"], g[f"c{d}"]
    assert rel(on.exact_sums(x, f, n_f, d, "type1", -1), g[f"t1dft_{d}"]) < 1e-13
    assert rel(on.exact_sums(x, c, n_f, d, "type2", +1), g[f"t2dft_{d}"]) < 1e-13
    assert tuple(on.plan(n_f, 1e-10)) == tuple(g[f"plan_{d}"])
    for eps in (1e-4, 1e-8, 1e-12):
        tag = f"{d}_{int(-np.log10(eps))}"
        a1 = on.type1(x, f, n_f, d, eps, -1, method="grid")
        a2 = on.type2(x, c, n_f, d, eps, +1, method="grid")
        # same algorithm; numpy FFT vs the reference's radix-2/3/5 FFT (roundoff only)
        assert rel(a1, g[f"t1grid_{tag}"]) < 1e-12
        assert rel(a2, g[f"t2grid_{tag}"]) < 1e-12
        # NUFFT contract vs exact sums
        assert rel(a1, g[f"t1dft_{d}"]) < eps
        assert rel(a2, g[f"t2dft_{d}"]) < eps


def tree_inputs(gen):
    import importlib.util
    spec = importlib.util.spec_from_file_location("mg", os.path.join(GOLD, "make_golden.py"))
    # make_golden imports the reference at module import; replicate only its generators
    src = open(spec.origin).read()
    start = src.index("def tree_inputs")
    ns = {"np": np}
    exec(src[start:src.index("def trees")], ns)
    return ns["tree_inputs"](gen)


TREES = {"cfg1": ("uniform2", 100, 1e-3, 1e-6, False),
         "clust3d": ("clust3", 40, 1e-4, 1e-9, False),
         "periodic2d": ("uniform2p", 50, 1e-4, 1e-8, True),
         "shell3d": ("shell3", 10, 1e-5, 1e-6, False)}


@pytest.mark.parametrize("name", list(TREES))
def test_tree_bit_exact_vs_reference(name):
    gen, n_s, delta, eps, periodic = TREES[name]
    y, x, _ = tree_inputs(gen)
    t = ot.build(y, x, n_s, delta, eps, periodic=periodic)
    g = load(f"tree_{name}.npz")
    assert t.l_c == int(g["l_c"]) and t.R == float(g["R"])
    assert np.array_equal(t.root_center, g["root_center"]) and t.root_side == float(g["root_side"])
    for f in ("level", "parent", "children", "coords", "is_leaf", "src_start", "src_count",
              "tgt_start", "tgt_count", "n_points"):
        assert np.array_equal(getattr(t, f), g[f]), f
    assert np.array_equal(t.src_perm, g["src_perm"]) and np.array_equal(t.tgt_perm, g["tgt_perm"])


def test_alg2_config1_vs_reference_primitives():
    y, x, q = tree_inputs("uniform2")
    g = load("alg2_cfg1.npz")
    u = ofgt.fgt_points(y, q, x, 1e-3, 1e-6, 100)
    assert rel(u, g["u"]) < 1e-12          # same algorithm on the reference primitives
    assert rel(u, g["exact"]) <= 10 * 1e-6  # SPEC.md:425 accuracy bar
    assert rel(g["u"], g["exact"]) <= 10 * 1e-6


# ------------------------------------------------------------------ volume (Alg 3/4)
def test_poly1d_vs_reference():
    from oracle import volume as ov
    g = load("poly1d.npz")
    t = np.linspace(-3, 3, 61)
    for lam in (1 / 64, 1 / 32, 1 / 16, 1 / 8, 0.25, 0.64):
        ref = g[f"J_{lam:.6f}"]
        got = ov.gauss_J(lam, 15, t)
        # relative to the table scale lam*sqrt(pi) (poly1d.py:181)
        assert np.max(np.abs(got - ref)) < 1e-11 * lam * np.sqrt(np.pi)
    tI = np.linspace(-100, 100, 401)
    assert np.max(np.abs(ov.fourier_I(23, tI) - g["I"])) < 1e-14
    b = ov.Basis(12)
    assert np.allclose(b.nodes, g["nodes12"], atol=1e-15, rtol=0)
    assert np.allclose(b.v2p, g["v2p12"], atol=1e-14, rtol=0)
    assert ov.tail_error(g["tail_c"]) == float(g["tail"])


def sigma_f(d):
    C = np.array([[0.1, -0.05, 0.02][:d], [-0.2, 0.15, -0.1][:d]])
    W, A = [0.05, 0.1], [1.0, 0.7]
    return (lambda p: sum(a * np.exp(-np.sum((p - c) ** 2, axis=-1) / w ** 2)
                          for c, w, a in zip(C, W, A))), C, W, A


@pytest.mark.parametrize("d,k,eps", [(2, 10, 1e-9), (3, 6, 1e-7)])
def test_density_tree_vs_reference(d, k, eps):
    from oracle import volume as ov
    g = load(f"dtree_{d}d.npz")
    t = ov.density_tree(sigma_f(d)[0], d, k, eps)
    for f in ("level", "parent", "children", "coords", "is_leaf"):
        assert np.array_equal(getattr(t, f), g[f]), f
    V = np.stack([t.values[b] for b in g["leaves"]]).reshape(len(g["leaves"]), -1)
    assert np.allclose(V.sum(axis=1), g["vsum"], rtol=1e-13, atol=1e-13)
    assert np.allclose((V * V).sum(axis=1), g["vsq"], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("d,k,delta,eps", [(1, 12, 1e-3, 1e-9), (2, 10, 1e-3, 1e-8),
                                           (3, 6, 1e-2, 1e-5)])
def test_volume_oracle_closed_form(d, k, delta, eps):
    """SPEC.md:651 acceptance 7(a): sum-of-Gaussians density, closed-form convolution."""
    from oracle import volume as ov
    dens, C, W, A = sigma_f(d)
    t = ov.density_tree(dens, d, k, eps * 0.1)
    u = ov.fgt_box(t, delta, eps)
    num = den = 0.0
    for b, ub in u.items():
        ex = ov.gaussian_box_convolution(t.leaf_points(b), delta, C, W, A)
        num += np.sum((ub - ex) ** 2)
        den += np.sum(ex ** 2)
    assert np.sqrt(num / den) <= 10 * eps


def test_volume_oracle_constant_density():
    """SPEC.md:259 / acceptance 7(c): sigma = 1 -> product of erf differences."""
    from scipy.special import erf
    from oracle import volume as ov
    t = ov.density_tree(lambda p: np.ones(p.shape[:-1]), 2, 8, 1e-10)
    delta, eps = 1e-2, 1e-9
    u = ov.fgt_box(t, delta, eps)
    for b, ub in u.items():
        x = t.leaf_points(b)
        ex = np.prod(np.sqrt(np.pi * delta) / 2 * (erf((0.5 - x) / np.sqrt(delta))
                                                   + erf((0.5 + x) / np.sqrt(delta))), axis=-1)
        assert np.max(np.abs(ub - ex)) <= 10 * eps * np.max(np.abs(ex))
