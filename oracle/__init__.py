"""Double-precision CPU oracle for the NURBS-Diff hot path (ctypes over nurbs_oracle.c).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The product package
``paper_2104_14547_b200`` never imports it and shares no code with it.

Every function follows a cited passage of /root/reference/PAPER.md (see nurbs_oracle.c);
inputs are fp32 arrays cast exactly to fp64 (R19 of DESIGN.md §3), outputs are fp64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nurbs_oracle.c")
_LIB = os.path.join(_HERE, "libnurbs_oracle.so")

REF_OK, REF_E_ARG, REF_E_KNOTS, REF_E_DOMAIN, REF_E_WEIGHT = 0, 1, 3, 4, 5


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, i32 = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)
        c_int = ctypes.c_int
        L.nurbs_ref_find_span.argtypes = [c_int, c_int, d, ctypes.c_double]
        L.nurbs_ref_find_span.restype = c_int
        L.nurbs_ref_basis_funs.argtypes = [c_int, ctypes.c_double, c_int, d, d]
        L.nurbs_ref_basis_funs.restype = None
        L.nurbs_ref_basis_dense.argtypes = [c_int, c_int, d, ctypes.c_double, d]
        L.nurbs_ref_basis_dense.restype = None
        L.nurbs_ref_check_knots.argtypes = [c_int, c_int, d]
        L.nurbs_ref_spans.argtypes = [c_int, c_int, d, c_int, d, i32, d]
        surf = [c_int] * 8 + [d, d, d, d, d]
        L.nurbs_ref_surface_fwd.argtypes = surf + [d]
        L.nurbs_ref_surface_bwd.argtypes = surf + [d, d]
        L.nurbs_ref_surface_bwd_eq89.argtypes = surf + [d, d]
        L.nurbs_ref_surface_bwd_selected.argtypes = surf + [d, c_int, i32, i32, i32, d]
        L.nurbs_ref_surface_dense.argtypes = [c_int] * 6 + [d, d, d, d, d, d, d]
        L.nurbs_ref_basis_ders1.argtypes = [c_int, ctypes.c_double, c_int, d, d]
        L.nurbs_ref_basis_ders1.restype = None
        L.nurbs_ref_surface_derivs.argtypes = surf + [d, d, d]
        pts = [c_int] * 7 + [d, d, d, d]
        L.nurbs_ref_surface_fwd_points.argtypes = pts + [d]
        L.nurbs_ref_surface_bwd_points.argtypes = pts + [d, d]
        L.nurbs_ref_basis_dknot.argtypes = [c_int, c_int, d, ctypes.c_double, c_int, d]
        L.nurbs_ref_basis_dknot.restype = None
        L.nurbs_ref_surface_knot_grad.argtypes = surf + [d, d, d]
        L.nurbs_ref_curve_knot_grad.argtypes = [c_int] * 5 + [d, d, d, d, d]
        L.nurbs_ref_curve_fwd.argtypes = [c_int] * 5 + [d, d, d, d]
        L.nurbs_ref_curve_bwd.argtypes = [c_int] * 5 + [d, d, d, d, d]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def cores() -> int:
    """Host threads the oracle may use (the process's CPU affinity, else os.cpu_count())."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def pmap(fn, items, threads: int | None = None) -> list:
    """[fn(*it) for it in items] on a pool of host threads, results in item order.

    The C oracle is called through ctypes, which releases the GIL, so the calls run in
    parallel (SURVEY.md §8(c) "Threading": threads over surfaces or u-row blocks; callers
    combine partial results in item order, so the result does not depend on the thread
    count)."""
    from concurrent.futures import ThreadPoolExecutor
    items = list(items)
    threads = threads or cores()
    if threads <= 1 or len(items) <= 1:
        return [fn(*it) for it in items]
    with ThreadPoolExecutor(max_workers=min(threads, len(items))) as ex:
        return list(ex.map(lambda it: fn(*it), items))


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _pi(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _chk(st: int, what: str):
    if st != REF_OK:
        raise OracleError(f"{what}: oracle status {st}")


def find_span(n: int, p: int, U, u: float) -> int:
    U = _d(U)
    return int(lib().nurbs_ref_find_span(n, p, _p(U), float(u)))


def basis_funs(s: int, u: float, p: int, U) -> np.ndarray:
    U = _d(U)
    N = np.zeros(p + 1)
    lib().nurbs_ref_basis_funs(s, float(u), p, _p(U), _p(N))
    return N


def basis_dense(n: int, p: int, U, u: float) -> np.ndarray:
    U = _d(U)
    N = np.zeros(n)
    lib().nurbs_ref_basis_dense(n, p, _p(U), float(u), _p(N))
    return N


def basis_ders1(s: int, u: float, p: int, U) -> np.ndarray:
    """First derivatives of the p+1 non-zero basis functions at span s (NEXT-3)."""
    U = _d(U)
    dN = np.zeros(p + 1)
    lib().nurbs_ref_basis_ders1(s, float(u), p, _p(U), _p(dN))
    return dN


def surface_derivs(ctrl, U, V, u, v, p: int, q: int, knots_batched: bool = False):
    """(S, S_u, S_v) each [B][n_u][n_v][3] by Eq.7 and its v analogue."""
    ctrl, U, V, u, v, dims = _surf_args(ctrl, U, V, u, v, p, q, knots_batched)
    B, n_u, n_v = dims[0], dims[5], dims[6]
    out, ou, ov = (np.zeros((B, n_u, n_v, 3)) for _ in range(3))
    _chk(lib().nurbs_ref_surface_derivs(*dims, _p(ctrl), _p(U), _p(V), _p(u), _p(v), _p(out), _p(ou), _p(ov)),
         "surface_derivs")
    return out, ou, ov


def spans(n: int, p: int, U, s) -> tuple[np.ndarray, np.ndarray]:
    U, s = _d(U), _d(s)
    sp = np.zeros(len(s), dtype=np.int32)
    N = np.zeros((len(s), p + 1))
    _chk(lib().nurbs_ref_spans(n, p, _p(U), len(s), _p(s), _pi(sp), _p(N)), "spans")
    return sp, N


def _surf_args(ctrl, U, V, u, v, p, q, knots_batched):
    ctrl = _d(ctrl)
    B, n, m, four = ctrl.shape
    assert four == 4
    U, V, u, v = _d(U), _d(V), _d(u), _d(v)
    return ctrl, U, V, u, v, (B, n, m, p, q, len(u), len(v), int(knots_batched))


def surface_fwd(ctrl, U, V, u, v, p: int, q: int, knots_batched: bool = False) -> np.ndarray:
    ctrl, U, V, u, v, dims = _surf_args(ctrl, U, V, u, v, p, q, knots_batched)
    B, n, m, _, _, n_u, n_v, _ = dims
    out = np.zeros((B, n_u, n_v, 3))
    _chk(lib().nurbs_ref_surface_fwd(*dims, _p(ctrl), _p(U), _p(V), _p(u), _p(v), _p(out)), "surface_fwd")
    return out


def surface_bwd(ctrl, U, V, u, v, gout, p: int, q: int, knots_batched: bool = False,
                form: str = "E") -> np.ndarray:
    """Gradient [B][n][m][4] = dL/d(x,y,z,w). form='E' (default) is the literal Eq.8 /
    Eq.9 sum; form='H' the homogeneous rewrite, pinned equal to it."""
    ctrl, U, V, u, v, dims = _surf_args(ctrl, U, V, u, v, p, q, knots_batched)
    B, n, m = dims[:3]
    g = _d(gout)
    assert g.shape == (B, dims[5], dims[6], 3)
    grad = np.zeros((B, n, m, 4))
    fn = lib().nurbs_ref_surface_bwd if form == "H" else lib().nurbs_ref_surface_bwd_eq89
    _chk(fn(*dims, _p(ctrl), _p(U), _p(V), _p(u), _p(v), _p(g), _p(grad)), "surface_bwd")
    return grad


def surface_bwd_selected(ctrl, U, V, u, v, gout, p, q, sel, knots_batched=False) -> np.ndarray:
    """Eq.8/9 gradient at selected control points sel = [(k, i, j), ...] -> [len(sel)][4]."""
    ctrl, U, V, u, v, dims = _surf_args(ctrl, U, V, u, v, p, q, knots_batched)
    g = _d(gout)
    sel = np.asarray(sel, dtype=np.int32).reshape(-1, 3)
    order = np.lexsort((sel[:, 2], sel[:, 1], sel[:, 0]))  # group by surface (spans cached per k)
    ss = np.ascontiguousarray(sel[order])
    k, i, j = (np.ascontiguousarray(ss[:, c]) for c in range(3))
    out = np.zeros((len(ss), 4))
    _chk(lib().nurbs_ref_surface_bwd_selected(*dims, _p(ctrl), _p(U), _p(V), _p(u), _p(v), _p(g),
                                              len(ss), _pi(k), _pi(i), _pi(j), _p(out)), "bwd_selected")
    res = np.zeros_like(out)
    res[order] = out
    return res


def surface_dense(ctrl2d, U, V, u, v, p, q, jacobian: bool = False):
    """Brute force on one surface: (out [n_u][n_v][3], J or None)."""
    ctrl = _d(ctrl2d)
    n, m, _ = ctrl.shape
    U, V, u, v = _d(U), _d(V), _d(u), _d(v)
    out = np.zeros((len(u), len(v), 3))
    J = np.zeros((len(u) * len(v) * 3, n * m * 4)) if jacobian else None
    _chk(lib().nurbs_ref_surface_dense(n, m, p, q, len(u), len(v), _p(ctrl), _p(U), _p(V), _p(u), _p(v),
                                       _p(out), _p(J) if jacobian else None), "surface_dense")
    return out, J


def _pts_args(ctrl, U, V, uv, p, q, knots_batched):
    ctrl, U, V, uv = _d(ctrl), _d(U), _d(V), _d(uv)
    B, n, m, four = ctrl.shape
    assert four == 4 and uv.shape[0] == B and uv.shape[2] == 2
    return ctrl, U, V, uv, (B, n, m, p, q, uv.shape[1], int(knots_batched))


def surface_fwd_points(ctrl, U, V, uv, p: int, q: int, knots_batched: bool = False) -> np.ndarray:
    """Paired points (NEXT-1): out [B][N][3] at uv [B][N][2] (Eq.3 per point)."""
    ctrl, U, V, uv, dims = _pts_args(ctrl, U, V, uv, p, q, knots_batched)
    out = np.zeros((dims[0], dims[5], 3))
    _chk(lib().nurbs_ref_surface_fwd_points(*dims, _p(ctrl), _p(U), _p(V), _p(uv), _p(out)), "fwd_points")
    return out


def surface_bwd_points(ctrl, U, V, uv, gout, p: int, q: int, knots_batched: bool = False) -> np.ndarray:
    """Paired points (NEXT-1): grad [B][n][m][4] by the literal Eq.8/9 (Form E)."""
    ctrl, U, V, uv, dims = _pts_args(ctrl, U, V, uv, p, q, knots_batched)
    g = _d(gout)
    assert g.shape == (dims[0], dims[5], 3)
    grad = np.zeros((dims[0], dims[1], dims[2], 4))
    _chk(lib().nurbs_ref_surface_bwd_points(*dims, _p(ctrl), _p(U), _p(V), _p(uv), _p(g), _p(grad)),
         "bwd_points")
    return grad


def basis_dknot(n: int, p: int, U, u: float, kk: int) -> np.ndarray:
    """dN_{i,p}(u)/dU[kk] for i = 0..n-1 (NEXT-4; Eq.4 differentiated)."""
    U = _d(U)
    dN = np.zeros(n)
    lib().nurbs_ref_basis_dknot(n, p, _p(U), float(u), int(kk), _p(dN))
    return dN


def surface_knot_grad(ctrl, U, V, u, v, gout, p: int, q: int, knots_batched: bool = False):
    """(dL/dU, dL/dV): [(B if batched else 1)][n+p+1], [..][m+q+1] (NEXT-4)."""
    ctrl, U, V, u, v, dims = _surf_args(ctrl, U, V, u, v, p, q, knots_batched)
    B, n, m = dims[:3]
    g = _d(gout)
    nb_ = B if knots_batched else 1
    gU, gV = np.zeros((nb_, n + p + 1)), np.zeros((nb_, m + q + 1))
    _chk(lib().nurbs_ref_surface_knot_grad(*dims, _p(ctrl), _p(U), _p(V), _p(u), _p(v), _p(g), _p(gU), _p(gV)),
         "surface_knot_grad")
    return gU, gV


def curve_knot_grad(ctrl, U, u, gout, p: int, knots_batched: bool = False) -> np.ndarray:
    ctrl, U, u, g = _d(ctrl), _d(U), _d(u), _d(gout)
    B, n, _ = ctrl.shape
    gU = np.zeros((B if knots_batched else 1, n + p + 1))
    _chk(lib().nurbs_ref_curve_knot_grad(B, n, p, len(u), int(knots_batched), _p(ctrl), _p(U), _p(u), _p(g),
                                         _p(gU)), "curve_knot_grad")
    return gU


def curve_fwd(ctrl, U, u, p: int, knots_batched: bool = False) -> np.ndarray:
    ctrl, U, u = _d(ctrl), _d(U), _d(u)
    B, n, _ = ctrl.shape
    out = np.zeros((B, len(u), 3))
    _chk(lib().nurbs_ref_curve_fwd(B, n, p, len(u), int(knots_batched), _p(ctrl), _p(U), _p(u), _p(out)),
         "curve_fwd")
    return out


def curve_bwd(ctrl, U, u, gout, p: int, knots_batched: bool = False) -> np.ndarray:
    ctrl, U, u, g = _d(ctrl), _d(U), _d(u), _d(gout)
    B, n, _ = ctrl.shape
    grad = np.zeros((B, n, 4))
    _chk(lib().nurbs_ref_curve_bwd(B, n, p, len(u), int(knots_batched), _p(ctrl), _p(U), _p(u), _p(g),
                                   _p(grad)), "curve_bwd")
    return grad
