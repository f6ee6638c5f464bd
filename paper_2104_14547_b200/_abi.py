"""ctypes declarations of the C ABI in include/nurbs.h (argument marshalling only).

The shared library ``libnurbs_b200.so`` is built in-tree by ``__graft_entry__.build()``
(or ``python -m paper_2104_14547_b200.build``). There is no fallback: importing the
binding without the library raises, so a missing CUDA path fails loudly.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NURBS_B200_LIB_EXPERIMENT") or os.path.join(HERE, "libnurbs_b200.so")

NURBS_OK = 0
NURBS_PATH_NO_TMA, NURBS_PATH_TC = 1, 2
NURBS_MAX_DEGREE = 5
STATUS_NAMES = {0: "NURBS_OK", 1: "NURBS_E_ARG", 2: "NURBS_E_UNSUPPORTED", 3: "NURBS_E_KNOTS",
                4: "NURBS_E_DOMAIN", 5: "NURBS_E_WEIGHT", 6: "NURBS_E_UNSORTED", 7: "NURBS_E_CUDA",
                8: "NURBS_E_WORKSPACE", 9: "NURBS_E_TABLES"}

# every symbol include/nurbs.h declares (checked by tests/test_abi_exports.py)
EXPORTS = ["nurbs_tables_bytes", "nurbs_tables", "nurbs_surface_fwd", "nurbs_surface_bwd",
           "nurbs_surface_bwd_workspace_bytes", "nurbs_curve_fwd", "nurbs_curve_bwd",
           "nurbs_curve_bwd_workspace_bytes", "nurbs_validate", "nurbs_strerror",
           "nurbs_surface_fit_step", "nurbs_surface_fit_workspace_bytes", "nurbs_surface_derivs",
           "nurbs_last_error_detail", "nurbs_abi_version", "nurbs_surface_points_fwd",
           "nurbs_surface_points_bwd", "nurbs_surface_points_bwd_workspace_bytes", "nurbs_validate_points",
           "nurbs_surface_bwd_knots", "nurbs_surface_bwd_knots_workspace_bytes", "nurbs_curve_bwd_knots",
           "nurbs_curve_bwd_knots_workspace_bytes", "nurbs_grid_plan", "nurbs_sum_partials", "nurbs_set_path_flags"]


class nurbs_shape(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("n", ctypes.c_int32), ("m", ctypes.c_int32),
                ("p", ctypes.c_int32), ("q", ctypes.c_int32), ("n_u", ctypes.c_int32),
                ("n_v", ctypes.c_int32), ("knots_batched", ctypes.c_int32)]


class NurbsError(RuntimeError):
    def __init__(self, status: int, detail: str, call: str):
        self.status = status
        super().__init__(f"{call}: {STATUS_NAMES.get(status, status)}: {detail}")


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    P, S, I = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    sh = ctypes.POINTER(nurbs_shape)
    sig = {
        "nurbs_tables_bytes": ([sh], S),
        "nurbs_tables": ([sh, P, P, P, P, P, P], I),
        "nurbs_surface_fwd": ([sh, P, P, P, P, P, P, P, P], I),
        "nurbs_surface_bwd": ([sh, P, P, P, P, P, P, P, P, P, P, P, S, P], I),
        "nurbs_surface_bwd_workspace_bytes": ([sh], S),
        "nurbs_curve_fwd": ([sh, P, P, P, P, P, P], I),
        "nurbs_curve_bwd": ([sh, P, P, P, P, P, P, P, P, S, P], I),
        "nurbs_curve_bwd_workspace_bytes": ([sh], S),
        "nurbs_validate": ([sh, P, P, P, P, P, P], I),
        "nurbs_surface_fit_step": ([sh, P, P, P, P, P, P, P, ctypes.c_float, P, P, P, S, P], I),
        "nurbs_surface_fit_workspace_bytes": ([sh], S),
        "nurbs_surface_derivs": ([sh, P, P, P, P, P, P, P, P, P, P], I),
        "nurbs_surface_points_fwd": ([sh, P, P, P, P, P, P], I),
        "nurbs_surface_points_bwd": ([sh, P, P, P, P, P, P, P, P, P, S, P], I),
        "nurbs_surface_points_bwd_workspace_bytes": ([sh], S),
        "nurbs_validate_points": ([sh, P, P, P, P, P], I),
        "nurbs_surface_bwd_knots": ([sh, P, P, P, P, P, P, P, P, P, P, P, S, P], I),
        "nurbs_surface_bwd_knots_workspace_bytes": ([sh], S),
        "nurbs_curve_bwd_knots": ([sh, P, P, P, P, P, P, P, P, S, P], I),
        "nurbs_curve_bwd_knots_workspace_bytes": ([sh], S),
        "nurbs_strerror": ([I], ctypes.c_char_p),
        "nurbs_last_error_detail": ([], ctypes.c_char_p),
        "nurbs_abi_version": ([], I),
        "nurbs_grid_plan": ([sh, ctypes.POINTER(ctypes.c_int32)], I),
        "nurbs_sum_partials": ([P, ctypes.c_int32, ctypes.c_int64, P, P], I),
        "nurbs_set_path_flags": ([I], I),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("NURBS_B200_LIB_EXPERIMENT") and not hasattr(L, name):
            continue  # an older experiment library (A/B timing) may lack newer entry points
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def check(status: int, call: str) -> None:
    if status != NURBS_OK:
        detail = load().nurbs_last_error_detail().decode(errors="replace")
        raise NurbsError(status, detail, call)
