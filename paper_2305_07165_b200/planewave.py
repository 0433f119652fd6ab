"""Host-side plane-wave parameters (Thm 2.1 of arXiv 2305.07165).

These feed the GPU tree (cutoff level, root side) and the plane-wave kernels (h, n_f,
weights), so they are evaluated with the same float64 numpy expressions as the
reference /root/reference/pkg/src/fgt/planewave.py (clamp :23-25, D0 :28-30,
pw_params :73-98) and tree.cutoff_level (/root/reference/pkg/src/fgt/tree.py:24-50):
identical inputs give bit-identical l_c, root side and box centres.
"""

from dataclasses import dataclass, field

import numpy as np

EPS_MIN = 1e-14
EPS_MAX = 0.1
EPS_CLAMP_HI = 0.099
MAX_LEVEL = 30
# one image layer reproduces the periodic kernel below this variance (planewave.py:20)
PERIODIC_IMAGE_DELTA = 1.0 / 36.0


def clamp_tolerance(epsilon):
    """Clamp epsilon into the supported window [1e-14, 0.099]."""
    e = float(epsilon)
    if e < EPS_MIN:
        e = EPS_MIN
    return min(e, EPS_CLAMP_HI)


def cutoff_factor(epsilon):
    """D0 = sqrt(log(3/eps)): beyond D0*sqrt(delta) the Gaussian is below eps."""
    return np.sqrt(np.log(3.0 / epsilon))


@dataclass(frozen=True)
class PwQuadrature:
    """Trapezoidal plane-wave rule for exp(-|x|^2/delta) on |x_i| <= R sqrt(delta).

    Modes m = -n_f/2 .. n_f/2-1 per axis, frequencies k_m = m h / sqrt(delta); the
    weights are stored pre-multiplied, w_m = h/(2 sqrt(pi)) exp(-m^2 h^2 / 4).
    """

    epsilon: float
    delta: float
    D0: float
    R: float
    h: float
    n_f: int
    dim: int
    weights_1d: np.ndarray = field(repr=False)

    @property
    def modes(self):
        return np.arange(-(self.n_f // 2), self.n_f // 2)

    @property
    def n_modes_total(self):
        return self.n_f ** self.dim

    def freqs_1d(self):
        return self.modes * self.h / np.sqrt(self.delta)

    def weights_tensor(self):
        out = self.weights_1d
        for _ in range(self.dim - 1):
            out = np.multiply.outer(out, self.weights_1d)
        return out


def pw_params(epsilon, delta, R=None, dim=1):
    """Plane-wave quadrature for tolerance epsilon and variance delta (R >= D0)."""
    eps = float(epsilon)
    if eps < EPS_MIN or eps >= EPS_MAX:
        raise ValueError(f"unsupported tolerance {eps:g}; need 1e-14 <= eps < 0.1")
    if not delta > 0:
        raise ValueError("delta must be positive")
    if dim not in (1, 2, 3):
        raise ValueError("dim must be 1, 2, or 3")
    D0 = cutoff_factor(eps)
    R = 2.0 * D0 if R is None else R
    if R < D0 * (1.0 - 1e-12):
        raise ValueError(f"range factor R={R:g} below D0={D0:g}; theorem requires R >= D0")
    h = 2.0 * np.pi / (R + D0)
    half = int(np.ceil(D0 * (R + D0) / np.pi))
    m = np.arange(-half, half)
    w = (h / (2.0 * np.sqrt(np.pi))) * np.exp(-(m * h) ** 2 / 4.0)
    return PwQuadrature(epsilon=eps, delta=float(delta), D0=D0, R=float(R), h=h,
                        n_f=2 * half, dim=dim, weights_1d=w)


def cutoff_level(delta, epsilon, L0=1.0, kind="density"):
    """(l_c, R) for a point tree over extent L0 or a fixed-root (density/periodic) tree."""
    if delta <= 0 or L0 < 0:
        raise ValueError("delta and L0 must be positive")
    D0 = cutoff_factor(clamp_tolerance(epsilon))
    cut = D0 * np.sqrt(delta)
    if kind == "point":
        if L0 <= cut:
            return 0, 2.0 * D0
        return min(int(np.ceil(np.log2(L0 / cut) - 1e-12)), MAX_LEVEL), 2.0 * D0
    if kind == "density":
        l_c = min(max(0, int(np.ceil(np.log2(L0 / (2.0 * cut)) - 1e-12))), MAX_LEVEL)
        s = L0 / 2 ** l_c
        return l_c, max(2.0 * s / np.sqrt(delta), D0)
    raise ValueError(f"unknown tree kind {kind!r}")


@dataclass(frozen=True)
class PeriodicSeries:
    """Truncated Fourier series of the periodic Gaussian on the unit cell:
    G_p(x) ~= sum_{|n| <= n_p} coeffs[n + n_p] exp(2 pi i n x), coeffs = sqrt(pi delta)
    exp(-(pi sqrt(delta) n)^2), n_p = ceil(sqrt(log(1/eps)) / (pi sqrt(delta)))
    (planewave.periodic_params, /root/reference/pkg/src/fgt/planewave.py:148-155)."""

    epsilon: float
    delta: float
    n_p: int
    coeffs: np.ndarray = field(repr=False)


def periodic_params(epsilon, delta):
    if epsilon <= 0 or delta <= 0:
        raise ValueError("epsilon and delta must be positive")
    n_p = int(np.ceil(np.sqrt(np.log(1.0 / epsilon)) / (np.pi * np.sqrt(delta))))
    n = np.arange(-n_p, n_p + 1)
    c = np.sqrt(np.pi * delta) * np.exp(-(np.pi * np.sqrt(delta) * n) ** 2)
    return PeriodicSeries(float(epsilon), float(delta), n_p, c)

