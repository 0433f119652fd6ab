"""Kernel backend of the B200 build (mirror of /root/reference/pkg/src/fgt/backend.py).

The reference binds its hot kernels once at import from the compiled module
`fgt._kernels_cy` (backend.py:17-27).  Here the compiled module is the CUDA library,
exposed through `_kernels_cuda`; there is deliberately no numpy fallback and no
FGT_FORCE_PYTHON switch on the product path — a missing library raises.
"""

from . import _kernels_cuda as _impl

BACKEND = _impl.BACKEND

gauss_direct = _impl.gauss_direct
gauss_direct_periodic = _impl.gauss_direct_periodic
nufft_spread = _impl.nufft_spread
nufft_interp = _impl.nufft_interp


def get_backends():
    """{name: module} of the available kernel backends (reference backend.py:30-38)."""
    return {"cuda": _impl}
