"""Periodic transform in the root Fourier-series regime (cutoff level <= 1, PAPER.md:1449-1453,
SPEC.md:411): one box (the unit cell), the periodic Gaussian's truncated Fourier series
 as its plane-wave expansion, no near field."""
import numpy as np
import pytest

from oracle import point_fgt as ofgt


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


CASES = [  # d, n, delta, eps
    (1, 3000, 0.05, 1e-9),
    (2, 4000, 0.03, 1e-8),
    (2, 3000, 0.02, 1e-12),   # delta < 1/36 but cutoff level <= 1
    (3, 3000, 0.1, 1e-6),
    (3, 2000, 0.04, 1e-10),
]


@pytest.mark.parametrize("case", CASES)
def test_oracle_root_series_vs_periodic_kernel(case):
    """The oracle's series evaluation against exact sums of the periodic kernel (the
    K-row image / Fourier forms, pinned to the reference's golden vectors)."""
    d, n, delta, eps = case
    r = np.random.default_rng(31)
    y = r.uniform(-0.5, 0.5, (400, d))
    x = r.uniform(-0.5, 0.5, (300, d))
    q = r.uniform(-1, 1, 400)
    u = ofgt.fgt_points_periodic_root(y, q, x, delta, eps)
    ex = ofgt.direct_oracle(y, q, x, delta, "periodic")
    assert rel(u, ex) <= eps


def test_params_select_root_series():
    from paper_2305_07165_b200.planewave import periodic_params
    from paper_2305_07165_b200.point_fgt import FgtParams
    p = FgtParams(3, 0.1, 1e-6, 50, True)
    s = periodic_params(1e-6, 0.1)
    assert p.root_series and p.tp.periodic == 2 and p.pw.n_f == 2 * s.n_p + 1
    assert np.allclose(p.pw.h / np.sqrt(0.1), 2 * np.pi)
    assert np.array_equal(p._w, s.coeffs)
    q = FgtParams(2, 1e-4, 1e-8, 50, True)
    assert not q.root_series and q.tp.periodic == 1


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["auto", "spread", "direct"])
@pytest.mark.parametrize("case", CASES)
def test_gpu_root_series(cuda, case, mode, monkeypatch):
    from paper_2305_07165_b200 import fgt_points
    if mode != "auto":
        monkeypatch.setenv("FGT_NUFFT_MODE", mode)
    d, n, delta, eps = case
    r = np.random.default_rng(32)
    y = r.uniform(-0.5, 0.5, (n, d))
    x = r.uniform(-0.5, 0.5, (n, d))
    q = r.uniform(-1, 1, n)
    u = fgt_points(y, q, x, delta, eps, 50, "periodic")
    ref = ofgt.fgt_points_periodic_root(y, q, x, delta, eps)
    assert rel(u, ref) <= 10 * eps
    sub = r.choice(n, size=300, replace=False)
    ex = ofgt.direct_oracle(y, q, x[sub], delta, "periodic")
    assert rel(u[sub], ex) <= 10 * eps
    # periodicity: a lattice translation leaves the potentials unchanged
    shift = np.zeros(d)
    shift[0] = 1.0
    us = fgt_points(y + shift, q, x - shift, delta, eps, 50, "periodic")
    assert rel(us, u) <= 10 * eps
