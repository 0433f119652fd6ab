"""B200-native (sm_100a) plane-wave fast Gauss transform (arXiv 2305.07165).

Public surface mirrors the reference package `fgt` (/root/reference/pkg/src/fgt):
`BACKEND`, the kernel backend module, `planewave` parameters, `tree.build_point_tree`,
and the discrete transform `fgt_points`.
"""

from .backend import BACKEND
from .point_fgt import fgt_points, fgt_points_device

__version__ = "0.1.0"

__all__ = ["BACKEND", "fgt_points", "fgt_points_device", "__version__"]
