"""Seeded generators of BASELINE.json's five configurations (SURVEY.md §8(d) recipes).

All inputs are synthetic (numpy default_rng, draws in the listed order, coordinates float64
C-order); no dataset is involved.  Shared by bench.py, tools/run_config.py and the
full-size parity tests.
"""

import numpy as np

CONFIGS = {
    1: dict(d=2, N=20_000, M=20_000, delta=1e-3, eps=1e-6, n_s=100, boundary="free"),
    2: dict(d=3, N=1_000_000, M=1_000_000, delta=1e-4, eps=1e-9, n_s=200, boundary="free"),
    3: dict(d=2, N=10_000_000, M=10_000_000, delta=1e-5, eps=1e-8, n_s=100, boundary="periodic"),
    5: dict(d=3, N=100_000_000, M=100_000_000, delta=1e-6, eps=1e-6, n_s=256, boundary="free"),
}

WORKLOADS = {
    1: "config1: discrete free-space FGT, d=2, N=M=2e4 uniform (targets = sources), delta=1e-3, eps=1e-6, s=100",
    2: ("config2: discrete free-space FGT, d=3, N=M=1e6, sources 8 Gaussian clusters (sigma=0.02, "
        "clipped), uniform targets, delta=1e-4, eps=1e-9, s=200"),
    3: "config3: discrete periodic FGT, d=2, N=M=1e7 uniform, delta=1e-5, eps=1e-8, s=100",
    5: ("config5: discrete free-space FGT, d=3, N=M=1e8, sources on a spherical shell r=0.35 "
        "thickness 1e-3, uniform targets, delta=1e-6, eps=1e-6, s=256"),
}


def config1(N=20_000):
    r = np.random.default_rng(0)
    y = r.uniform(-0.5, 0.5, (N, 2))
    return y, r.uniform(-1, 1, N), y.copy()


def config2(N=1_000_000, M=None):
    M = N if M is None else M
    r = np.random.default_rng(1)
    C = r.uniform(-0.5, 0.5, (8, 3))
    lab = r.integers(0, 8, N)
    y = np.clip(C[lab] + 0.02 * r.standard_normal((N, 3)), -0.5, 0.5)
    q = r.standard_normal(N)
    x = np.random.default_rng(2).uniform(-0.5, 0.5, (M, 3))
    return y, q, x


def config3(N=10_000_000, M=None):
    M = N if M is None else M
    r = np.random.default_rng(0)
    y = r.uniform(-0.5, 0.5, (N, 2))
    q = r.uniform(-1, 1, N)
    return y, q, np.random.default_rng(1).uniform(-0.5, 0.5, (M, 2))


def config5(N=100_000_000, M=None):
    """Thin spherical shell (r = 0.35, thickness 1e-3) sources, uniform targets.  The
    recipe's expressions are applied in place (same roundings as y = rho * u / |u|)."""
    M = N if M is None else M
    r = np.random.default_rng(0)
    y = r.standard_normal((N, 3))
    y /= np.linalg.norm(y, axis=1, keepdims=True)
    rho = 0.35 + 1e-3 * (r.uniform(size=N) - 0.5)
    y *= rho[:, None]
    del rho
    q = r.uniform(-1, 1, N)
    x = np.random.default_rng(1).uniform(-0.5, 0.5, (M, 3))
    return y, q, x


def generate(cfg_id, N=None, M=None):
    cfg = CONFIGS[cfg_id]
    N = cfg["N"] if N is None else int(N)
    if cfg_id == 1:
        return config1(N)
    fn = {2: config2, 3: config3, 5: config5}[cfg_id]
    return fn(N, M)
