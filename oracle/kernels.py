"""Oracle: the four backend kernels (restates /root/reference/pkg/src/fgt/_kernels_py.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np

ROWS = 1024


def gauss_sum(targets, sources, charges, inv_delta, r2_cut, out, periodic=False):
    """_kernels_py.gauss_direct / gauss_direct_periodic (:14-46): accumulate into out."""
    targets = np.atleast_2d(targets)
    sources = np.atleast_2d(sources)
    for a in range(0, targets.shape[0], ROWS):
        b = min(a + ROWS, targets.shape[0])
        diff = targets[a:b, None, :] - sources[None, :, :]
        if periodic:
            diff = diff - np.round(diff)
        r2 = (diff * diff).sum(axis=-1)
        with np.errstate(under="ignore"):
            g = np.exp(-r2 * inv_delta)
        if np.isfinite(r2_cut):
            g = np.where(r2 > r2_cut, 0.0, g)
        out[a:b] += g @ charges
    return out


def _taps(x, n_r, m_sp, tau):
    """_kernels_py._spread_weights (:49-62): nearest index and Gaussian tap weights."""
    hr = 2.0 * np.pi / n_r
    base = np.rint(x / hr).astype(np.int64)
    o = np.arange(-m_sp, m_sp + 1)
    z = x[:, :, None] - (base[:, :, None] + o) * hr
    with np.errstate(under="ignore"):
        return base, np.exp(-z * z / (4.0 * tau)), o


def _tensor_taps(base, w, o, n_r, sl):
    d = base.shape[1]
    wt = w[sl, 0, :]
    ix = (base[sl, 0, None] + o) % n_r
    for k in range(1, d):
        wt = (wt[:, :, None] * w[sl, k, None, :]).reshape(wt.shape[0], -1)
        ik = (base[sl, k, None] + o) % n_r
        ix = (ix[:, :, None] * n_r + ik[:, None, :]).reshape(ix.shape[0], -1)
    return wt, ix


def spread(x, values, n_r, m_sp, tau, grid):
    """_kernels_py.nufft_spread (:65-81)."""
    base, w, o = _taps(x, n_r, m_sp, tau)
    flat = grid.reshape(-1)
    for a in range(0, x.shape[0], ROWS):
        sl = slice(a, min(a + ROWS, x.shape[0]))
        wt, ix = _tensor_taps(base, w, o, n_r, sl)
        np.add.at(flat, ix, wt * values[sl, None])
    return grid


def interp(x, grid, n_r, m_sp, tau):
    """_kernels_py.nufft_interp (:84-100)."""
    base, w, o = _taps(x, n_r, m_sp, tau)
    flat = grid.reshape(-1)
    out = np.empty(x.shape[0], dtype=np.complex128)
    for a in range(0, x.shape[0], ROWS):
        sl = slice(a, min(a + ROWS, x.shape[0]))
        wt, ix = _tensor_taps(base, w, o, n_r, sl)
        out[sl] = (wt * flat[ix]).sum(axis=1)
    return out
