"""Oracle: type-1/type-2 NUFFT (restates /root/reference/pkg/src/fgt/nufft.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The FFT is numpy's (the reference
uses its own unnormalised radix-2/3/5 FFT, fftpack.py:69-84; same transform).
"""

import numpy as np

from . import kernels


def smooth(n):
    """fftpack.next_smooth (fftpack.py:30-35)."""
    m = max(int(n), 1)
    while True:
        k = m
        for r in (2, 3, 5):
            while k % r == 0:
                k //= r
        if k == 1:
            return m
        m += 1


def modes(n_f):
    return np.arange(n_f) - n_f // 2


def exact_sums(points, data, n_f, dim, kind, sign):
    """nufft.dft_oracle (nufft.py:65-103): tensor-factored exact sums."""
    pts = np.asarray(points, dtype=float).reshape(-1, dim)
    m = modes(n_f)
    if kind == "type1":
        out = np.zeros((n_f,) * dim, dtype=np.complex128)
        step = max(1, 2 ** 22 // n_f ** dim)
        for a in range(0, pts.shape[0], step):
            E = [np.exp(sign * 1j * np.outer(pts[a:a + step, k], m)) for k in range(dim)]
            f = np.asarray(data[a:a + step], dtype=np.complex128)
            if dim == 1:
                out += E[0].T @ f
            elif dim == 2:
                out += (E[0] * f[:, None]).T @ E[1]
            else:
                out += np.einsum("ja,jb,jc->abc", E[0] * f[:, None], E[1], E[2])
        return out
    coeffs = np.asarray(data, dtype=np.complex128).reshape((n_f,) * dim)
    out = np.empty(pts.shape[0], dtype=np.complex128)
    step = max(1, 2 ** 22 // n_f ** max(dim - 1, 1))
    for a in range(0, pts.shape[0], step):
        E = [np.exp(sign * 1j * np.outer(pts[a:a + step, k], m)) for k in range(dim)]
        if dim == 1:
            out[a:a + step] = E[0] @ coeffs
        elif dim == 2:
            out[a:a + step] = np.einsum("jb,jb->j", E[0] @ coeffs, E[1])
        else:
            t = np.einsum("ja,abc->jbc", E[0], coeffs)
            t = np.einsum("jbc,jb->jc", t, E[1])
            out[a:a + step] = np.einsum("jc,jc->j", t, E[2])
    return out


def plan(n_f, epsilon):
    """nufft._plan (nufft.py:106-115): grid size, half-width, Gaussian variance."""
    epsilon = max(float(epsilon), 1e-14)
    w = int(np.ceil(np.log(30.0 / epsilon) / (np.pi / np.sqrt(2.0)))) + 1
    n_r = smooth(2 * n_f)
    if 2 * w + 1 > n_r:
        n_r = smooth(max(2 * n_f, 2 * w + 2))
    tau = np.pi * w / (n_r * np.sqrt(n_r * (n_r - n_f)))
    return n_r, w, tau


def prefers_direct(n_f, dim, M, w):
    """nufft._use_direct (nufft.py:118-121)."""
    size = n_f ** dim
    spread_cost = M * (2 * w + 1) ** dim
    fft_cost = size * max(np.log2(max(size, 2)), 1.0)
    return M * size < 4 * (fft_cost + spread_cost + size)


def _deconv(n_f, dim, n_r, tau):
    """nufft._deconv_tensor (nufft.py:124-131)."""
    m = modes(n_f)
    rho = (np.sqrt(np.pi / tau) / n_r) * np.exp(m * m * tau)
    out = rho
    for _ in range(dim - 1):
        out = np.multiply.outer(out, rho)
    return out


def _fftn(a, sign):
    # unnormalised sum_j a_j exp(sign 2 pi i jk/n)
    return np.fft.fftn(a) if sign < 0 else np.fft.ifftn(a) * a.size


def type1(points, strengths, n_f, dim, epsilon, sign=-1, method=None):
    """nufft.nufft_type1 (nufft.py:139-162)."""
    pts = np.asarray(points, dtype=float).reshape(-1, dim)
    f = np.asarray(strengths, dtype=np.complex128)
    if pts.shape[0] == 0:
        return np.zeros((n_f,) * dim, dtype=np.complex128)
    n_r, w, tau = plan(n_f, epsilon)
    if method == "direct" or (method is None and prefers_direct(n_f, dim, pts.shape[0], w)):
        return exact_sums(pts, f, n_f, dim, "type1", sign)
    x = np.mod(pts, 2.0 * np.pi)
    grid = np.zeros((n_r,) * dim, dtype=np.complex128)
    kernels.spread(x, f, n_r, w, tau, grid)
    D = _fftn(grid, -1)
    b = np.mod(-sign * modes(n_f), n_r)
    F = D[np.ix_(*[b] * dim)]
    return F * _deconv(n_f, dim, n_r, tau)


def type2(points, coeffs, n_f, dim, epsilon, sign=+1, method=None):
    """nufft.nufft_type2 (nufft.py:165-183)."""
    pts = np.asarray(points, dtype=float).reshape(-1, dim)
    c = np.asarray(coeffs, dtype=np.complex128).reshape((n_f,) * dim)
    if pts.shape[0] == 0:
        return np.zeros(0, dtype=np.complex128)
    n_r, w, tau = plan(n_f, epsilon)
    if method == "direct" or (method is None and prefers_direct(n_f, dim, pts.shape[0], w)):
        return exact_sums(pts, c, n_f, dim, "type2", sign)
    x = np.mod(pts, 2.0 * np.pi)
    E = np.zeros((n_r,) * dim, dtype=np.complex128)
    b = np.mod(-sign * modes(n_f), n_r)
    E[np.ix_(*[b] * dim)] = c * _deconv(n_f, dim, n_r, tau)
    return kernels.interp(x, _fftn(E, -1), n_r, w, tau)
