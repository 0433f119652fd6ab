"""ctypes binding of libfgtcuda.so (C ABI in include/fgt_cuda.h).

There is no CPU fallback: if the library is missing or cannot be loaded, importing the
CUDA paths raises immediately (FgtLibraryError) instead of silently computing on the
host.
"""

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# FGT_LIB_PATH selects an alternative build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("FGT_LIB_PATH") or os.path.join(HERE, "libfgtcuda.so")

FGT_OK, FGT_EINVAL, FGT_ECUDA, FGT_ERANGE, FGT_ENOMEM = 0, 1, 2, 3, 4


class FgtLibraryError(RuntimeError):
    """libfgtcuda.so is missing or failed to load."""


class FgtPwParams(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n_f", ctypes.c_int32), ("delta", ctypes.c_double),
                ("D0", ctypes.c_double), ("h", ctypes.c_double),
                ("weights_1d", ctypes.POINTER(ctypes.c_double))]


class FgtTreeParams(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("periodic", ctypes.c_int32), ("n_s", ctypes.c_int64),
                ("D0", ctypes.c_double), ("delta", ctypes.c_double),
                ("l_c_periodic", ctypes.c_int32), ("part_rank", ctypes.c_int32),
                ("part_size", ctypes.c_int32)]


class FgtTreeInfo(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("l_c", ctypes.c_int32), ("n_levels", ctypes.c_int32),
                ("periodic", ctypes.c_int32), ("n_boxes", ctypes.c_int64),
                ("n_leaves", ctypes.c_int64), ("n_dense", ctypes.c_int64),
                ("n_sources", ctypes.c_int64), ("n_targets", ctypes.c_int64),
                ("root_center", ctypes.c_double * 3), ("root_side", ctypes.c_double)]


class FgtListInfo(ctypes.Structure):
    _fields_ = [("n_p_entries", ctypes.c_int64), ("n_d_entries", ctypes.c_int64),
                ("n_psi_boxes", ctypes.c_int64), ("n_direct_pairs", ctypes.c_int64)]


class FgtPhaseTimes(ctypes.Structure):
    _fields_ = ([(n, ctypes.c_double) for n in
                 ("tree_ms", "lists_ms", "form_ms", "gather_ms", "eval_ms", "direct_ms",
                  "total_ms", "h2d_ms", "d2h_ms")] + [("launches", ctypes.c_int64)]
                + [(n, ctypes.c_double) for n in
                   ("k_form_ms", "k_gather_ms", "k_eval_ms", "k_direct_ms")]
                + [(n, ctypes.c_int64) for n in
                   ("n_boxes", "n_dense", "n_psi", "n_src_dense", "n_tgt_psi", "n_p_entries",
                    "n_direct_pairs", "n_modes", "n_spread_boxes", "n_src_spread",
                    "n_spread_psi", "n_tgt_spread")]
                + [("nufft_w", ctypes.c_int32), ("nufft_G", ctypes.c_int32)])

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_PI64 = ctypes.POINTER(ctypes.c_int64)
_PD = ctypes.POINTER(ctypes.c_double)


class FgtBoxPlan(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("k", ctypes.c_int32), ("n_f", ctypes.c_int32),
                ("n_levels", ctypes.c_int32), ("l_c", ctypes.c_int32),
                ("n_leaves", ctypes.c_int64), ("n_pw", ctypes.c_int64),
                ("val2pw", _PD), ("pw2val", _PD), ("n_rows", ctypes.c_int64), ("rows", _PD),
                ("n_tables", ctypes.c_int64), ("dtab", _PD),
                ("n_form", ctypes.c_int64), ("form_leaf", _PI64), ("form_pw", _PI64),
                ("form_level", _PI64),
                ("n_stages", ctypes.c_int64), ("n_dst", ctypes.c_int64),
                ("n_entries", ctypes.c_int64), ("stage_off", _PI64), ("stage_kind", _PI64),
                ("dst", _PI64), ("dst_acc", _PI64), ("dst_off", _PI64), ("ent_src", _PI64),
                ("ent_rows", _PI64),
                ("n_eval", ctypes.c_int64), ("eval_leaf", _PI64), ("eval_pw", _PI64),
                ("eval_level", _PI64),
                ("n_dpairs", ctypes.c_int64), ("d_tgt", _PI64), ("d_src", _PI64),
                ("d_tab", _PI64)]


_P = ctypes.c_void_p
_D = ctypes.c_double
_I64 = ctypes.c_int64
_I = ctypes.c_int

# name -> (restype, argtypes); also the list the CPU test checks against the header.
class FgtInterpTree(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("k", ctypes.c_int32), ("periodic", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("n_leaves", ctypes.c_int64),
                ("level", ctypes.POINTER(ctypes.c_int32)), ("coords", ctypes.POINTER(ctypes.c_int64)),
                ("coeffs", ctypes.POINTER(ctypes.c_double)), ("root_low", ctypes.c_double * 3),
                ("root_side", ctypes.c_double)]


SIGNATURES = {
    "fgt_box_interp": (ctypes.c_int, [ctypes.POINTER(FgtInterpTree), ctypes.c_void_p, ctypes.c_int64,
                                      ctypes.c_void_p]),
    "fgt_box_interp_dev": (ctypes.c_int, [ctypes.POINTER(FgtInterpTree), ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "fgt_last_error": (ctypes.c_char_p, []),
    "fgt_version": (ctypes.c_char_p, []),
    "fgt_launch_count": (_I64, []),
    "fgt_reset_launch_count": (None, []),
    "fgt_gauss_direct": (_I, [_P, _I64, _P, _I64, _P, _I, _D, _D, _I, _P]),
    "fgt_nufft_spread": (_I, [_P, _I64, _I, _P, _I64, _I, _D, _P]),
    "fgt_nufft_interp": (_I, [_P, _I64, _I, _P, _I64, _I, _D, _P]),
    "fgt_gauss_direct_dev": (_I, [_P, _I64, _P, _I64, _P, _I, _D, _D, _I, _P, _P]),
    "fgt_nufft_spread_dev": (_I, [_P, _I64, _I, _P, _I64, _I, _D, _P, _P]),
    "fgt_nufft_interp_dev": (_I, [_P, _I64, _I, _P, _I64, _I, _D, _P, _P]),
    "fgt_tree_build_dev": (_I, [_P, _I64, _P, _I64, ctypes.POINTER(FgtTreeParams), _P,
                                ctypes.POINTER(_P)]),
    "fgt_tree_get_info": (_I, [_P, ctypes.POINTER(FgtTreeInfo)]),
    "fgt_tree_copy_out": (_I, [_P] + [_P] * 12),
    "fgt_tree_free": (None, [_P]),
    "fgt_tree_lists": (_I, [_P, ctypes.POINTER(FgtListInfo)]),
    "fgt_tree_copy_lists": (_I, [_P] + [_P] * 6),
    "fgt_points_dev": (_I, [_P, _I64, _P, _P, _I64, ctypes.POINTER(FgtTreeParams),
                            ctypes.POINTER(FgtPwParams), _P, _P, ctypes.POINTER(FgtPhaseTimes)]),
    "fgt_points_begin": (_I, [_P, _I64, _P, _P, _I64, ctypes.POINTER(FgtTreeParams),
                              ctypes.POINTER(FgtPwParams), _P, ctypes.POINTER(_P)]),
    "fgt_points_exchange_counts": (_I, [_P, _P, _P, ctypes.POINTER(_I64)]),
    "fgt_points_pack": (_I, [_P, _P]),
    "fgt_points_unpack": (_I, [_P, _P]),
    "fgt_points_finish": (_I, [_P, _P, ctypes.POINTER(FgtPhaseTimes)]),
    "fgt_points_run_free": (None, [_P]),
    "fgt_points": (_I, [_P, _I64, _P, _P, _I64, ctypes.POINTER(FgtTreeParams),
                        ctypes.POINTER(FgtPwParams), _P, ctypes.POINTER(FgtPhaseTimes)]),
    "fgt_bench_fp64_peak": (_I, [_I, ctypes.POINTER(_D)]),
    "fgt_partition_bounds": (_I, [_P, _I64, ctypes.c_int32, _P]),
    "fgt_box_dev": (_I, [ctypes.POINTER(FgtBoxPlan), _P, _P, _P, ctypes.POINTER(FgtPhaseTimes)]),
    "fgt_box": (_I, [ctypes.POINTER(FgtBoxPlan), _P, _P, ctypes.POINTER(FgtPhaseTimes)]),
    "fgt_box_tail_dev": (_I, [_P, _I64, _I, _I, _P, _P, _P, _P, _P]),
    "fgt_box_tail": (_I, [_P, _I64, _I, _I, _P, _P, _P, _P]),
    "fgt_box_nodes_dev": (_I, [_P, _P, _I64, _I, _I, _P, _P, _D, _P, _P]),
    "fgt_box_balance_flags": (_I, [_P, _P, _P, _I64, _I, _I, _P]),
    "fgt_box_retain": (_I, [ctypes.POINTER(FgtBoxPlan), _P, _P, ctypes.POINTER(FgtPhaseTimes),
                            ctypes.POINTER(_P)]),
    "fgt_box_refine": (_I, [_P, ctypes.POINTER(FgtBoxPlan), _P, ctypes.POINTER(FgtPhaseTimes)]),
    "fgt_box_state_free": (_I, [_P]),
}

_lib = None


def load():
    """Load (once) and return the ctypes handle; raise FgtLibraryError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FgtLibraryError(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as e:
        raise FgtLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status):
    """Map a C status code to the reference's Python exceptions."""
    if status == FGT_OK:
        return
    msg = load().fgt_last_error().decode(errors="replace")
    if status in (FGT_EINVAL, FGT_ERANGE):
        raise ValueError(msg)
    if status == FGT_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def ptr(a):
    """Raw data pointer of a C-contiguous numpy array (or None)."""
    if a is None:
        return None
    return ctypes.c_void_p(a.ctypes.data)


def as_c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)
