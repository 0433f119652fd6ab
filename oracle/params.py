"""Oracle: plane-wave parameters (restates /root/reference/pkg/src/fgt/planewave.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

from dataclasses import dataclass

import numpy as np


def clamp_eps(epsilon):
    """planewave.clamp_tolerance (planewave.py:23-25)."""
    return min(max(float(epsilon), 1e-14), 0.099)


def d0_of(epsilon):
    """planewave.cutoff_factor (planewave.py:28-30)."""
    return np.sqrt(np.log(3.0 / epsilon))


@dataclass(frozen=True)
class Quad:
    """planewave.PwQuadrature (planewave.py:33-70)."""

    D0: float
    R: float
    h: float
    n_f: int
    dim: int
    delta: float
    w1: np.ndarray

    @property
    def m(self):
        return np.arange(self.n_f) - self.n_f // 2

    def wtensor(self):
        w = self.w1
        for _ in range(self.dim - 1):
            w = np.multiply.outer(w, self.w1)
        return w


def quad(epsilon, delta, R=None, dim=1):
    """planewave.pw_params (planewave.py:73-98)."""
    eps = float(epsilon)
    if not (1e-14 <= eps < 0.1):
        raise ValueError("unsupported tolerance")
    if delta <= 0:
        raise ValueError("delta must be positive")
    D0 = d0_of(eps)
    if R is None:
        R = 2.0 * D0
    if R < D0 * (1.0 - 1e-12):
        raise ValueError("R < D0")
    h = 2.0 * np.pi / (R + D0)
    M = int(np.ceil(D0 * (R + D0) / np.pi))
    m = np.arange(-M, M)
    w1 = (h / (2.0 * np.sqrt(np.pi))) * np.exp(-(m * h) ** 2 / 4.0)
    return Quad(D0=D0, R=float(R), h=h, n_f=2 * M, dim=dim, delta=float(delta), w1=w1)


def periodic_np(epsilon, delta):
    """planewave.periodic_params n_p (planewave.py:130-155)."""
    return int(np.ceil(np.sqrt(np.log(1.0 / epsilon)) / (np.pi * np.sqrt(delta))))


def cut_level(delta, epsilon, L0=1.0, kind="density"):
    """tree.cutoff_level (tree.py:24-50)."""
    D0 = d0_of(clamp_eps(epsilon))
    cut = D0 * np.sqrt(delta)
    if kind == "point":
        if L0 <= cut:
            return 0, 2.0 * D0
        return min(int(np.ceil(np.log2(L0 / cut) - 1e-12)), 30), 2.0 * D0
    l_c = min(max(0, int(np.ceil(np.log2(L0 / (2.0 * cut)) - 1e-12))), 30)
    s = L0 / 2 ** l_c
    return l_c, max(2.0 * s / np.sqrt(delta), D0)


def periodic_kernel_1d(x, delta):
    """planewave._periodic_1d image/Fourier forms (planewave.py:158-171)."""
    x = x - np.round(x)
    with np.errstate(under="ignore"):
        if delta < 1.0 / 36.0:
            return np.exp(-x * x / delta) + np.exp(-(x + 1) ** 2 / delta) + np.exp(-(x - 1) ** 2 / delta)
        n_p = periodic_np(1e-16, delta)
        n = np.arange(1, n_p + 1)
        damp = np.exp(-(np.pi * np.sqrt(delta) * n) ** 2)
        return np.sqrt(np.pi * delta) * (1.0 + 2.0 * np.cos(2 * np.pi * np.multiply.outer(x, n)) @ damp)
