"""CUDA (sm_100a) implementations of the reference's hot kernels.

Drop-in for the compiled-backend slot ``fgt._kernels_cy`` that the reference declares
(/root/reference/pkg/setup.py:12-18) and binds in ``fgt.backend``
(/root/reference/pkg/src/fgt/backend.py:17-27).  Same call signatures, argument
meaning and in-place conventions as the numpy fallback
/root/reference/pkg/src/fgt/_kernels_py.py:14-100:

* ``gauss_direct`` / ``gauss_direct_periodic`` accumulate into ``out`` and return it;
* ``nufft_spread`` accumulates into the caller-zeroed ``grid_out`` and returns it;
* ``nufft_interp`` returns a new complex128 array.

All arithmetic runs in libfgtcuda.so (host pointers; H2D/D2H inside the call).
"""

import numpy as np

from . import _lib

BACKEND = "cuda"


def _accumulate(out, dtype, fn):
    """Run fn(buf) on a C-contiguous buffer aliasing `out` when possible."""
    if out.dtype == dtype and out.flags.c_contiguous and out.flags.writeable:
        fn(out)
    else:
        buf = np.ascontiguousarray(out, dtype=dtype)
        fn(buf)
        out[...] = buf
    return out


def _direct(targets, sources, charges, inv_delta, r2_cut, out, periodic):
    lib = _lib.load()
    t = np.atleast_2d(_lib.as_c(targets))
    s = np.atleast_2d(_lib.as_c(sources))
    q = _lib.as_c(charges).reshape(-1)
    nt, d = t.shape
    ns = s.shape[0] if s.size else 0
    if s.size and s.shape[1] != d:
        raise ValueError(f"sources have dimension {s.shape[1]}, targets {d}")
    if q.shape[0] != ns:
        raise ValueError("sources/charges length mismatch")
    if out.shape[0] != nt:
        raise ValueError("out length != number of targets")

    def run(buf):
        _lib.check(lib.fgt_gauss_direct(_lib.ptr(t), nt, _lib.ptr(s), ns, _lib.ptr(q), d,
                                        float(inv_delta), float(r2_cut), int(periodic),
                                        _lib.ptr(buf)))
    return _accumulate(out, np.float64, run)


def gauss_direct(targets, sources, charges, inv_delta, r2_cut, out):
    """out[i] += sum_j exp(-||targets[i]-sources[j]||^2 * inv_delta) * q_j (r2 <= r2_cut)."""
    return _direct(targets, sources, charges, inv_delta, r2_cut, out, periodic=False)


def gauss_direct_periodic(targets, sources, charges, inv_delta, r2_cut, out):
    """Minimum-image variant of gauss_direct on the unit cell."""
    return _direct(targets, sources, charges, inv_delta, r2_cut, out, periodic=True)


def nufft_spread(x, values, n_r, m_sp, tau, grid_out):
    """Scatter complex point values onto the periodic oversampled grid (in place)."""
    lib = _lib.load()
    xx = np.atleast_2d(_lib.as_c(x))
    M, d = xx.shape
    v = _lib.as_c(values, np.complex128).reshape(-1)
    if v.shape[0] != M:
        raise ValueError("points/values length mismatch")
    if grid_out.shape != (n_r,) * d:
        raise ValueError(f"grid_out shape {grid_out.shape} != {(n_r,) * d}")

    def run(buf):
        _lib.check(lib.fgt_nufft_spread(_lib.ptr(xx), M, d, _lib.ptr(v), int(n_r), int(m_sp),
                                        float(tau), _lib.ptr(buf)))
    return _accumulate(grid_out, np.complex128, run)


def nufft_interp(x, grid, n_r, m_sp, tau):
    """Gather values of a smooth periodic grid function at arbitrary points."""
    lib = _lib.load()
    xx = np.atleast_2d(_lib.as_c(x))
    M, d = xx.shape
    g = _lib.as_c(grid, np.complex128)
    if g.shape != (n_r,) * d:
        raise ValueError(f"grid shape {g.shape} != {(n_r,) * d}")
    out = np.empty(M, dtype=np.complex128)
    _lib.check(lib.fgt_nufft_interp(_lib.ptr(xx), M, d, _lib.ptr(g), int(n_r), int(m_sp),
                                    float(tau), _lib.ptr(out)))
    return out
