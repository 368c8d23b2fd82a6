"""ctypes binding of the C-ABI (include/dla.h) in libdla_b200.so.

The shared library is built in-tree (``paper_1710_08717_b200/libdla_b200.so``)
by ``__graft_entry__.build()`` / ``make -C paper_1710_08717_b200/csrc``.
There is no fallback: if the library is missing or fails to load, importing
the operator layer raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DLA_LIB_PATH: an alternative in-tree build of the same library (tuning A/B runs)
LIB_PATH = os.environ.get("DLA_LIB_PATH") or os.path.join(HERE, "libdla_b200.so")

_i64, _int, _vp, _sz = C.c_int64, C.c_int, C.c_void_p, C.c_size_t

DLA_OK = 0
STATUS_NAMES = {0: "OK", 1: "SHAPE", 2: "NOT_SPD", 3: "SINGULAR", 4: "CONVERGENCE", 5: "ALIAS",
                6: "ASYMMETRIC", 7: "CUDA", 8: "WORKSPACE", 9: "INVALID"}
OPS = {"gemm": 0, "gemm2": 1, "syrk": 2, "trmm": 3, "trsm": 4, "potrf": 5, "potri": 6,
       "sumlogdiag": 7, "gelqf": 8, "syevd": 9, "chol_chain": 10, "gesvd": 11}
WS_BACKWARD, WS_RIGHTSIDE = 1, 2

# argument kinds: P = device pointer, I = int64, F = flag (int), S = scalar (T), Z = size_t
_SIGS = {
    "gemm2_fwd": "IIIIPPPFFSPZP",
    "gemm_fwd": "IIIIPPPFFSSPZP",
    "gemm2_bwd": "IIIIPPPPPFFSPZP",
    "gemm_bwd": "IIIIPPPPPFFSSPZP",
    "syrk_fwd": "IIIPPFSPZP",
    "syrk_bwd": "IIIPPPFSPZP",
    "trmm_fwd": "IIIPPFFFSPZP",
    "trmm_into": "IIIPPPFFFSPZP",
    "trmm_bwd": "IIIPPPPPFFFSPZP",
    "trsm_fwd": "IIIPPFFFSPPZP",
    "trsm_bwd": "IIIPPPPPFFFSPZP",
    "potrf_fwd": "IIPFPPZP",
    "potrf_bwd": "IIPPPFPZP",
    "potri_fwd": "IIPFPPZP",
    "potri_into": "IIPPFPPZP",
    "potri_bwd": "IIPPPPFPZP",
    "sumlogdiag_fwd": "IIPPPZP",
    "sumlogdiag_bwd": "IIPPPFPZP",
    "gelqf_fwd": "IIIPPPPZP",
    "gelqf_bwd": "IIIPPPPPPZP",
    "syevd_fwd": "IIPPPPZP",
    "syevd_bwd": "IIPPPPPSPZP",
    "chol_chain_fwdbwd": "IIPPPPPPPZP",
    "gesvd_fwd": "IIIPPPPPZP",
    "gesvd_bwd": "IIIPPPPPPPSPPZP",
}


class _Lib:
    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise ImportError(
                f"libdla_b200.so not found at {path}: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        self.path = path
        self.lib = C.CDLL(path)
        L = self.lib
        L.dla_status_string.restype = C.c_char_p
        L.dla_status_string.argtypes = [_int]
        L.dla_version.restype = C.c_char_p
        L.dla_workspace_bytes.restype = _sz
        L.dla_workspace_bytes.argtypes = [_int, _int, _i64, _i64, _i64, _i64, _int]
        L.dla_info_check.restype = _int
        L.dla_info_check.argtypes = [_vp, _i64, _vp, C.POINTER(_i64), C.POINTER(_i64)]
        L.dla_launch_count.restype = C.c_longlong
        L.dla_launch_count.argtypes = []
        L.dla_prof_enable.restype = None
        L.dla_prof_enable.argtypes = [_int]
        L.dla_prof_read.restype = C.c_longlong
        L.dla_prof_read.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.dla_prof_read_max.restype = C.c_longlong
        L.dla_prof_read_max.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.dla_gp_rbf_ws_bytes.restype = _sz
        L.dla_gp_rbf_ws_bytes.argtypes = [_i64, _i64, _i64]
        gsig = [_i64, _i64, _i64, _vp, C.c_double, C.c_double, C.c_double]
        L.dla_gp_rbf_fwd_f64.argtypes = gsig + [_vp, _vp, _sz, _vp]
        L.dla_gp_rbf_fwd_f64.restype = _int
        L.dla_gp_rbf_bwd_f64.argtypes = gsig + [_vp, _vp, _vp, _vp, _sz, _vp]
        L.dla_gp_rbf_bwd_f64.restype = _int
        L.dla_gp_nll_assemble_f64.argtypes = [_i64, _i64, _vp, _vp, _vp, _vp]
        L.dla_gp_nll_assemble_f64.restype = _int
        L.dla_potrf_bwd_ws_bytes_f64.restype = _sz
        L.dla_potrf_bwd_ws_bytes_f64.argtypes = [_i64, _i64]
        L.dla_gp_potrf_inv_f64.argtypes = [_i64, _i64, _vp, _vp, _vp, _sz, _vp]
        L.dla_gp_potrf_inv_f64.restype = _int
        L.dla_potrf_bwd_begin_f64.argtypes = [_i64, _i64, _vp, _int, _vp, _sz, _vp]
        L.dla_potrf_bwd_begin_f64.restype = _int
        L.dla_potrf_bwd_end_f64.argtypes = [_i64, _i64, _vp, _vp, _vp, _int, _vp, _sz, _vp]
        L.dla_potrf_bwd_end_f64.restype = _int
        L.dla_ml_shift_copy_f64.argtypes = [_i64, _i64, _vp, _vp, C.c_double, _vp]
        L.dla_ml_shift_copy_f64.restype = _int
        L.dla_axpy_f64.argtypes = [_i64, C.c_double, _vp, _vp, _vp]
        L.dla_axpy_f64.restype = _int
        L.dla_ml_reduce_ws_bytes.restype = _sz
        L.dla_ml_reduce_ws_bytes.argtypes = [_i64]
        L.dla_ml_reduce_f64.argtypes = [_i64, _i64, _vp, _vp, _vp, C.c_double, _vp, _vp, _sz, _vp]
        L.dla_ml_reduce_f64.restype = _int
        L.dla_gp_pullback_ws_bytes.restype = _sz
        L.dla_gp_pullback_ws_bytes.argtypes = [_i64, _i64, _i64]
        L.dla_gp_rbf_bwd_sym_ws_bytes.restype = _sz
        L.dla_gp_rbf_bwd_sym_ws_bytes.argtypes = [_i64, _i64, _i64]
        L.dla_gp_pullback_f64.argtypes = [_i64, _i64, _i64, _vp, C.c_double, C.c_double, C.c_double, _vp, _vp, _vp,
                                          _vp, _vp, _sz, _vp, _sz, _vp]
        L.dla_gp_pullback_f64.restype = _int
        L.dla_potrf_inv_join_f64.argtypes = [_vp]
        L.dla_potrf_inv_join_f64.restype = _int
        for sfx in ("f32", "f64"):
            wsf = getattr(L, f"dla_kalman_ws_bytes_{sfx}")
            wsf.restype = _sz
            wsf.argtypes = [_i64, _i64, _i64, _i64]
            kf = getattr(L, f"dla_kalman_nll_fwdbwd_{sfx}")
            kf.argtypes = [_i64, _i64, _i64, _i64] + [_vp] * 7 + [_i64] + [_vp] * 9 + [_vp, _sz, _vp]
            kf.restype = _int
        self.fns = {}
        for name, sig in _SIGS.items():
            for suffix, scal in (("f32", C.c_float), ("f64", C.c_double)):
                f = getattr(L, f"dla_{name}_{suffix}")
                kinds = {"P": _vp, "I": _i64, "F": _int, "S": scal, "Z": _sz}
                f.argtypes = [kinds[k] for k in sig]
                f.restype = _int
                self.fns[(name, suffix)] = f

    def fn(self, name: str, suffix: str):
        return self.fns[(name, suffix)]


_LIB = None


def lib() -> _Lib:
    global _LIB
    if _LIB is None:
        _LIB = _Lib()
    return _LIB


def exported_symbols():
    """Every dla_* symbol include/dla.h declares (used by the CPU symbol test)."""
    names = ["dla_status_string", "dla_version", "dla_workspace_bytes", "dla_info_check",
             "dla_launch_count", "dla_prof_enable", "dla_prof_read", "dla_prof_read_max", "dla_gp_rbf_ws_bytes",
             "dla_gp_rbf_fwd_f64", "dla_gp_rbf_bwd_f64", "dla_gp_nll_assemble_f64",
             "dla_ml_shift_copy_f64", "dla_axpy_f64", "dla_ml_reduce_ws_bytes", "dla_ml_reduce_f64",
             "dla_potrf_bwd_ws_bytes_f64", "dla_potrf_inv_join_f64",
             "dla_potrf_bwd_begin_f64", "dla_potrf_bwd_end_f64", "dla_gp_potrf_inv_f64",
             "dla_kalman_ws_bytes_f32", "dla_kalman_ws_bytes_f64",
             "dla_kalman_nll_fwdbwd_f32", "dla_kalman_nll_fwdbwd_f64",
             "dla_tape_ew_ws_bytes", "dla_tape_ew_f32", "dla_tape_ew_f64",
             "dla_gp_rbf_bwd_sym_ws_bytes", "dla_gp_pullback_ws_bytes", "dla_gp_pullback_f64"]
    for name in _SIGS:
        for s in ("f32", "f64"):
            names.append(f"dla_{name}_{s}")
    return names
