"""Python binding of include/nurbs.h: same names as the C ABI, torch tensors as device
memory. Argument marshalling only — every step of the path runs in libnurbs_b200.so.

Low-level calls (``nurbs_surface_fwd`` ...) take a ``nurbs_shape`` and tensors (or raw
device addresses as ints) exactly like the C functions; ``stream`` defaults to torch's
current CUDA stream. Convenience wrappers (``surface_fwd`` ...) infer the shape and allocate
outputs with torch.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from ._abi import check, load, nurbs_shape

_F32 = torch.float32


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            raise ValueError("libnurbs_b200 takes device tensors (CUDA); got a CPU tensor")
        if not x.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return ctypes.c_void_p(x.data_ptr())
    if isinstance(x, Tables):
        return ctypes.c_void_p(x.buf.data_ptr())
    raise TypeError(f"cannot pass {type(x)} as a device pointer")


def _sizes(sh: nurbs_shape) -> dict:
    """Element counts every tensor argument must have for shape `sh` (include/nurbs.h)."""
    kb = sh.B if sh.knots_batched else 1
    curve = sh.m == 1 and sh.q == 0
    return {"ctrl": sh.B * sh.n * sh.m * 4, "U": kb * (sh.n + sh.p + 1),
            "V": None if curve else kb * (sh.m + sh.q + 1), "u": sh.n_u, "v": None if curve else sh.n_v,
            "pts": sh.B * sh.n_u * sh.n_v * 3}


def _expect(sh: nurbs_shape, exact: bool = False, **named):
    """Raise ValueError unless every tensor argument is float32 and holds the element count
    the shape implies: at least that many in the C-ABI mirrors (a smaller buffer would be read
    or written out of bounds; a larger one, e.g. a reused slot, is only partly used), exactly
    that many in the convenience wrappers. A float64 tensor would be reinterpreted, so dtype
    is always checked. Raw device addresses (ints) are the caller's responsibility, as in C.
    The keyword's prefix names its kind: ctrl, U, V, u, v or pts."""
    sz = _sizes(sh)
    for key, t in named.items():
        if not isinstance(t, torch.Tensor):
            continue
        kind = key.split("_")[0]
        if t.dtype != _F32:
            raise ValueError(f"{key}: expected float32, got {t.dtype}")
        want = sz[kind]
        if want is not None and (t.numel() != want if exact else t.numel() < want):
            raise ValueError(f"{key}: expected {want} elements for shape (B={sh.B}, n={sh.n}, m={sh.m}, "
                             f"p={sh.p}, q={sh.q}, n_u={sh.n_u}, n_v={sh.n_v}, "
                             f"knots_batched={sh.knots_batched}), got {t.numel()} {tuple(t.shape)}")


def _expect_tables(sh: nurbs_shape, tables):
    """Tables are built for one shape: refuse them for another (their offsets would be wrong)."""
    if isinstance(tables, Tables):
        a, b = tables.shape, sh
        fa = tuple(getattr(a, f) for f, _ in nurbs_shape._fields_ if f != "B")
        fb = tuple(getattr(b, f) for f, _ in nurbs_shape._fields_ if f != "B")
        if fa != fb or (a.knots_batched and a.B != b.B):
            raise ValueError(f"tables were built for (n, m, p, q, n_u, n_v, knots_batched) = {fa}, "
                             f"the call has {fb}")


def _stream(stream):
    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, torch.cuda.Stream):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


# ----------------------------------------------------------------------------- shapes
def surface_shape(ctrl: torch.Tensor, U: torch.Tensor, u: torch.Tensor, v: torch.Tensor,
                  p: int, q: int) -> nurbs_shape:
    B, n, m, four = ctrl.shape
    assert four == 4, "ctrl must be [B][n][m][4]"
    return nurbs_shape(B, n, m, p, q, u.numel(), v.numel(), 1 if U.dim() == 2 else 0)


def curve_shape(ctrl: torch.Tensor, U: torch.Tensor, u: torch.Tensor, p: int) -> nurbs_shape:
    B, n, four = ctrl.shape
    assert four == 4, "ctrl must be [B][n][4]"
    return nurbs_shape(B, n, 1, p, 0, u.numel(), 1, 1 if U.dim() == 2 else 0)


def _is_curve(sh: nurbs_shape) -> bool:
    return sh.m == 1 and sh.q == 0


def bwd_workspace_bytes(sh: nurbs_shape) -> int:
    L = load()
    f = L.nurbs_curve_bwd_workspace_bytes if _is_curve(sh) else L.nurbs_surface_bwd_workspace_bytes
    return int(f(ctypes.byref(sh)))


class path_flags:
    """Context manager selecting kernel paths (nurbs_set_path_flags), e.g.
    ``with path_flags(no_tma=True): ...`` runs the per-thread IO path and
    ``with path_flags(tc=True): ...`` the tensor-core backward; restores on exit."""

    def __init__(self, no_tma: bool = False, tc: bool = False):
        from ._abi import NURBS_PATH_NO_TMA, NURBS_PATH_TC
        self.flags = (NURBS_PATH_NO_TMA if no_tma else 0) | (NURBS_PATH_TC if tc else 0)

    def __enter__(self):
        self.prev = load().nurbs_set_path_flags(self.flags)
        return self

    def __exit__(self, *exc):
        load().nurbs_set_path_flags(self.prev)


def grid_plan(sh: nurbs_shape) -> dict:
    """The grid kernels' launch plan for `sh` (nurbs_grid_plan; host only)."""
    out = (ctypes.c_int32 * 6)()
    check(load().nurbs_grid_plan(ctypes.byref(sh), out), "nurbs_grid_plan")
    return dict(zip(("K", "row_blocks", "col_blocks", "band_rows", "direct", "ctas"), list(out)))


# ----------------------------------------------------------------------------- C ABI mirror
def nurbs_tables(sh, U, V, u, v, tables, stream=None):
    _expect(sh, U=U, V=V, u=u, v=v)
    check(load().nurbs_tables(ctypes.byref(sh), _ptr(U), _ptr(V), _ptr(u), _ptr(v), _ptr(tables),
                              _stream(stream)), "nurbs_tables")


def nurbs_surface_fwd(sh, ctrl, U, V, u, v, tables, out, stream=None):
    _expect(sh, ctrl=ctrl, U=U, V=V, u=u, v=v, pts_out=out)
    _expect_tables(sh, tables)
    check(load().nurbs_surface_fwd(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(V), _ptr(u), _ptr(v),
                                   _ptr(tables), _ptr(out), _stream(stream)), "nurbs_surface_fwd")


def nurbs_surface_bwd(sh, ctrl, U, V, u, v, tables, grad_out, grad_ctrl, grad_U, grad_V,
                      workspace, ws_bytes, stream=None):
    _expect(sh, ctrl=ctrl, U=U, V=V, u=u, v=v, pts_grad_out=grad_out, ctrl_grad=grad_ctrl, U_grad=grad_U,
            V_grad=grad_V)
    _expect_tables(sh, tables)
    check(load().nurbs_surface_bwd(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(V), _ptr(u), _ptr(v),
                                   _ptr(tables), _ptr(grad_out), _ptr(grad_ctrl), _ptr(grad_U),
                                   _ptr(grad_V), _ptr(workspace), ctypes.c_size_t(ws_bytes),
                                   _stream(stream)), "nurbs_surface_bwd")


def nurbs_curve_fwd(sh, ctrl, U, u, tables, out, stream=None):
    _expect(sh, ctrl=ctrl, U=U, u=u, pts_out=out)
    _expect_tables(sh, tables)
    check(load().nurbs_curve_fwd(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(u), _ptr(tables), _ptr(out),
                                 _stream(stream)), "nurbs_curve_fwd")


def nurbs_curve_bwd(sh, ctrl, U, u, tables, grad_out, grad_ctrl, grad_U, workspace, ws_bytes, stream=None):
    _expect(sh, ctrl=ctrl, U=U, u=u, pts_grad_out=grad_out, ctrl_grad=grad_ctrl, U_grad=grad_U)
    _expect_tables(sh, tables)
    check(load().nurbs_curve_bwd(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(u), _ptr(tables),
                                 _ptr(grad_out), _ptr(grad_ctrl), _ptr(grad_U), _ptr(workspace),
                                 ctypes.c_size_t(ws_bytes), _stream(stream)), "nurbs_curve_bwd")


def nurbs_surface_fit_step(sh, ctrl, U, V, u, v, tables, target, lr, grad_ctrl, loss, workspace, ws_bytes,
                           stream=None):
    _expect(sh, ctrl=ctrl, U=U, V=V, u=u, v=v, pts_target=target, ctrl_grad=grad_ctrl)
    _expect_tables(sh, tables)
    check(load().nurbs_surface_fit_step(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(V), _ptr(u), _ptr(v),
                                        _ptr(tables), _ptr(target), ctypes.c_float(lr), _ptr(grad_ctrl),
                                        _ptr(loss), _ptr(workspace), ctypes.c_size_t(ws_bytes), _stream(stream)),
          "nurbs_surface_fit_step")


def nurbs_surface_derivs(sh, ctrl, U, V, u, v, out, out_u, out_v, normals, stream=None):
    _expect(sh, ctrl=ctrl, U=U, V=V, u=u, v=v, pts_out=out, pts_u=out_u, pts_v=out_v, pts_normals=normals)
    check(load().nurbs_surface_derivs(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(V), _ptr(u), _ptr(v), _ptr(out),
                                      _ptr(out_u), _ptr(out_v), _ptr(normals), _stream(stream)),
          "nurbs_surface_derivs")


def surface_derivs(ctrl, U, V, u, v, p: int, q: int, with_points: bool = True, with_normals: bool = True,
                   stream=None):
    """(S or None, S_u, S_v, normals or None), each [B][n_u][n_v][3] (NEXT-3, Eq.7)."""
    sh = surface_shape(ctrl, U, u, v, p, q)
    mk = lambda: torch.empty((sh.B, sh.n_u, sh.n_v, 3), dtype=_F32, device=ctrl.device)
    out = mk() if with_points else None
    ou, ov = mk(), mk()
    nrm = mk() if with_normals else None
    nurbs_surface_derivs(sh, ctrl, U, V, u, v, out, ou, ov, nrm, stream)
    return out, ou, ov, nrm


def fit_workspace_bytes(sh: nurbs_shape) -> int:
    return int(load().nurbs_surface_fit_workspace_bytes(ctypes.byref(sh)))


def nurbs_sum_partials(parts, out, stream=None):
    """out[k] = sum over r (ascending) of parts[r][k] — the fixed-order sum of the per-rank
    partial gradients of a point-sharded backward (include/nurbs.h). parts: [R][n] float32."""
    if parts.dtype != _F32 or out.dtype != _F32 or parts.dim() != 2 or out.numel() != parts.shape[1]:
        raise ValueError(f"parts must be float32 [R][n] and out float32 [n]; got {tuple(parts.shape)}, {tuple(out.shape)}")
    check(load().nurbs_sum_partials(_ptr(parts), parts.shape[0], out.numel(), _ptr(out), _stream(stream)),
          "nurbs_sum_partials")


def nurbs_validate(sh, ctrl, U, V, u, v, stream=None):
    _expect(sh, ctrl=ctrl, U=U, V=V, u=u, v=v)
    check(load().nurbs_validate(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(V), _ptr(u), _ptr(v),
                                _stream(stream)), "nurbs_validate")


# ----------------------------------------------------------------------------- knot gradients (NEXT-4)
def knots_workspace_bytes(sh: nurbs_shape) -> int:
    L = load()
    f = L.nurbs_curve_bwd_knots_workspace_bytes if _is_curve(sh) else L.nurbs_surface_bwd_knots_workspace_bytes
    return int(f(ctypes.byref(sh)))


def nurbs_surface_bwd_knots(sh, ctrl, U, V, u, v, tables, grad_out, grad_ctrl, grad_U, grad_V, workspace, ws_bytes,
                            stream=None):
    _expect(sh, ctrl=ctrl, U=U, V=V, u=u, v=v, pts_grad_out=grad_out, ctrl_grad=grad_ctrl, U_grad=grad_U,
            V_grad=grad_V)
    _expect_tables(sh, tables)
    check(load().nurbs_surface_bwd_knots(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(V), _ptr(u), _ptr(v),
                                         _ptr(tables), _ptr(grad_out), _ptr(grad_ctrl), _ptr(grad_U), _ptr(grad_V),
                                         _ptr(workspace), ctypes.c_size_t(ws_bytes), _stream(stream)),
          "nurbs_surface_bwd_knots")


def nurbs_curve_bwd_knots(sh, ctrl, U, u, tables, grad_out, grad_ctrl, grad_U, workspace, ws_bytes, stream=None):
    _expect(sh, ctrl=ctrl, U=U, u=u, pts_grad_out=grad_out, ctrl_grad=grad_ctrl, U_grad=grad_U)
    _expect_tables(sh, tables)
    check(load().nurbs_curve_bwd_knots(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(u), _ptr(tables), _ptr(grad_out),
                                       _ptr(grad_ctrl), _ptr(grad_U), _ptr(workspace), ctypes.c_size_t(ws_bytes),
                                       _stream(stream)), "nurbs_curve_bwd_knots")


def surface_bwd_knots(ctrl, U, V, u, v, grad_out, p: int, q: int, tables=None, stream=None):
    """(grad_ctrl, dL/dU, dL/dV) with TRUE knot gradients (NEXT-4); dL/dU is [n+p+1] for
    shared knots (summed over the batch) or [B][n+p+1] for batched knots."""
    sh = surface_shape(ctrl, U, u, v, p, q)
    grad_ctrl = torch.empty_like(ctrl)
    gU, gV = torch.empty_like(U), torch.empty_like(V)
    ws = knots_workspace_bytes(sh)
    work = torch.empty(max(ws, 1), dtype=torch.uint8, device=ctrl.device)
    nurbs_surface_bwd_knots(sh, ctrl, U, V, u, v, tables, grad_out, grad_ctrl, gU, gV, work, ws, stream)
    return grad_ctrl, gU, gV


def curve_bwd_knots(ctrl, U, u, grad_out, p: int, tables=None, stream=None):
    sh = curve_shape(ctrl, U, u, p)
    grad_ctrl = torch.empty_like(ctrl)
    gU = torch.empty_like(U)
    ws = knots_workspace_bytes(sh)
    work = torch.empty(max(ws, 1), dtype=torch.uint8, device=ctrl.device)
    nurbs_curve_bwd_knots(sh, ctrl, U, u, tables, grad_out, grad_ctrl, gU, work, ws, stream)
    return grad_ctrl, gU


# ----------------------------------------------------------------------------- paired points (NEXT-1)
def points_shape(ctrl: torch.Tensor, U: torch.Tensor, uv: torch.Tensor, p: int, q: int) -> nurbs_shape:
    B, n, m, four = ctrl.shape
    assert four == 4, "ctrl must be [B][n][m][4]"
    assert uv.dim() == 3 and uv.shape[0] == B and uv.shape[2] == 2, "uv must be [B][N][2]"
    return nurbs_shape(B, n, m, p, q, uv.shape[1], 1, 1 if U.dim() == 2 else 0)


def points_workspace_bytes(sh: nurbs_shape) -> int:
    return int(load().nurbs_surface_points_bwd_workspace_bytes(ctypes.byref(sh)))


def _expect_points(sh, uv=None, exact: bool = False, **named):
    _expect(sh, exact, **named)
    if isinstance(uv, torch.Tensor) and (uv.dtype != _F32 or (uv.numel() != sh.B * sh.n_u * 2 if exact
                                                              else uv.numel() < sh.B * sh.n_u * 2)):
        raise ValueError(f"uv: expected float32 [B={sh.B}][N={sh.n_u}][2], got {uv.dtype} {tuple(uv.shape)}")


def nurbs_surface_points_fwd(sh, ctrl, U, V, uv, out, stream=None):
    _expect_points(sh, uv, ctrl=ctrl, U=U, V=V, pts_out=out)
    check(load().nurbs_surface_points_fwd(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(V), _ptr(uv), _ptr(out),
                                          _stream(stream)), "nurbs_surface_points_fwd")


def nurbs_surface_points_bwd(sh, ctrl, U, V, uv, grad_out, grad_ctrl, grad_U, grad_V, workspace, ws_bytes,
                             stream=None):
    _expect_points(sh, uv, ctrl=ctrl, U=U, V=V, pts_grad_out=grad_out, ctrl_grad=grad_ctrl, U_grad=grad_U,
                   V_grad=grad_V)
    check(load().nurbs_surface_points_bwd(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(V), _ptr(uv),
                                          _ptr(grad_out), _ptr(grad_ctrl), _ptr(grad_U), _ptr(grad_V),
                                          _ptr(workspace), ctypes.c_size_t(ws_bytes), _stream(stream)),
          "nurbs_surface_points_bwd")


def nurbs_validate_points(sh, ctrl, U, V, uv, stream=None):
    _expect_points(sh, uv, ctrl=ctrl, U=U, V=V)
    check(load().nurbs_validate_points(ctypes.byref(sh), _ptr(ctrl), _ptr(U), _ptr(V), _ptr(uv), _stream(stream)),
          "nurbs_validate_points")


def surface_points_fwd(ctrl, U, V, uv, p: int, q: int, out=None, stream=None):
    """S at paired points: out [B][N][3] for uv [B][N][2]."""
    sh = points_shape(ctrl, U, uv, p, q)
    _expect_points(sh, uv, True, ctrl=ctrl, U=U, V=V, pts_out=out)
    if out is None:
        out = torch.empty((sh.B, sh.n_u, 3), dtype=_F32, device=ctrl.device)
    nurbs_surface_points_fwd(sh, ctrl, U, V, uv, out, stream)
    return out


def surface_points_bwd(ctrl, U, V, uv, grad_out, p: int, q: int, grad_ctrl=None, grad_U=None, grad_V=None,
                       workspace=None, stream=None):
    """dL/d(x,y,z,w) [B][n][m][4] at paired points (deterministic)."""
    sh = points_shape(ctrl, U, uv, p, q)
    _expect_points(sh, uv, True, ctrl=ctrl, U=U, V=V, pts_grad_out=grad_out, ctrl_grad=grad_ctrl)
    if grad_ctrl is None:
        grad_ctrl = torch.empty_like(ctrl)
    ws = points_workspace_bytes(sh)
    if workspace is None and ws > 0:
        workspace = torch.empty(ws, dtype=torch.uint8, device=ctrl.device)
    nurbs_surface_points_bwd(sh, ctrl, U, V, uv, grad_out, grad_ctrl, grad_U, grad_V, workspace, ws, stream)
    return grad_ctrl


# ----------------------------------------------------------------------------- tables
@dataclass
class Tables:
    """Span/basis tables for fixed knots and a fixed parameter grid (P:171 precompute)."""
    shape: nurbs_shape
    buf: torch.Tensor

    @staticmethod
    def build(sh: nurbs_shape, U, V, u, v, stream=None) -> "Tables":
        nbytes = int(load().nurbs_tables_bytes(ctypes.byref(sh)))
        dev = (U if isinstance(U, torch.Tensor) else u).device
        buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        nurbs_tables(sh, U, V, u, v, buf, stream)
        return Tables(sh, buf)


# ----------------------------------------------------------------------------- wrappers
def surface_fwd(ctrl, U, V, u, v, p: int, q: int, tables: Tables | None = None, out=None, stream=None):
    sh = surface_shape(ctrl, U, u, v, p, q)
    _expect(sh, True, ctrl=ctrl, U=U, V=V, u=u, v=v, pts_out=out)
    if out is None:
        out = torch.empty((sh.B, sh.n_u, sh.n_v, 3), dtype=_F32, device=ctrl.device)
    nurbs_surface_fwd(sh, ctrl, U, V, u, v, tables, out, stream)
    return out


def surface_bwd(ctrl, U, V, u, v, grad_out, p: int, q: int, tables: Tables | None = None,
                grad_ctrl=None, grad_U=None, grad_V=None, workspace=None, stream=None):
    sh = surface_shape(ctrl, U, u, v, p, q)
    _expect(sh, True, ctrl=ctrl, U=U, V=V, u=u, v=v, pts_grad_out=grad_out, ctrl_grad=grad_ctrl, U_grad=grad_U,
            V_grad=grad_V)
    if grad_ctrl is None:
        grad_ctrl = torch.empty_like(ctrl)
    ws = bwd_workspace_bytes(sh)
    if workspace is None and ws > 0:
        workspace = torch.empty(ws, dtype=torch.uint8, device=ctrl.device)
    nurbs_surface_bwd(sh, ctrl, U, V, u, v, tables, grad_out, grad_ctrl, grad_U, grad_V, workspace, ws, stream)
    return grad_ctrl


def curve_fwd(ctrl, U, u, p: int, tables: Tables | None = None, out=None, stream=None):
    sh = curve_shape(ctrl, U, u, p)
    _expect(sh, True, ctrl=ctrl, U=U, u=u, pts_out=out)
    if out is None:
        out = torch.empty((sh.B, sh.n_u, 3), dtype=_F32, device=ctrl.device)
    nurbs_curve_fwd(sh, ctrl, U, u, tables, out, stream)
    return out


def curve_bwd(ctrl, U, u, grad_out, p: int, tables: Tables | None = None, grad_ctrl=None, grad_U=None,
              workspace=None, stream=None):
    sh = curve_shape(ctrl, U, u, p)
    _expect(sh, True, ctrl=ctrl, U=U, u=u, pts_grad_out=grad_out, ctrl_grad=grad_ctrl, U_grad=grad_U)
    if grad_ctrl is None:
        grad_ctrl = torch.empty_like(ctrl)
    ws = bwd_workspace_bytes(sh)
    if workspace is None and ws > 0:
        workspace = torch.empty(ws, dtype=torch.uint8, device=ctrl.device)
    nurbs_curve_bwd(sh, ctrl, U, u, tables, grad_out, grad_ctrl, grad_U, workspace, ws, stream)
    return grad_ctrl


class SurfaceFitter:
    """The fitting loop of §4.2: SGD on P and w of one batch of surfaces toward a
    target point grid, each iteration one fused step (nurbs_surface_fit_step). `run(iters)`
    records `iters` steps once into a CUDA graph (no host work per iteration) and replays it.
    Argument marshalling only: every iteration runs in libnurbs_b200's kernels."""

    def __init__(self, ctrl, U, V, u, v, target, p: int, q: int, lr: float, tables: "Tables | None" = None):
        self.ctrl, self.U, self.V, self.u, self.v, self.target = ctrl, U, V, u, v, target
        self.sh = surface_shape(ctrl, U, u, v, p, q)
        self.lr, self.tables = lr, tables
        self.grad = torch.empty_like(ctrl)
        self.ws_bytes = fit_workspace_bytes(self.sh)
        self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=ctrl.device)
        self.losses = None
        self._graph = None

    def step(self, loss_out, stream=None):
        nurbs_surface_fit_step(self.sh, self.ctrl, self.U, self.V, self.u, self.v, self.tables, self.target,
                               self.lr, self.grad, loss_out, self.ws, self.ws_bytes, stream)

    def run(self, iters: int, graph: bool = True) -> torch.Tensor:
        """Run `iters` steps; returns the per-iteration loss history (device tensor)."""
        if self.losses is None or self.losses.numel() != iters:
            self.losses = torch.zeros(iters, dtype=torch.float32, device=self.ctrl.device)
            self._graph = None
        if not graph:
            for k in range(iters):
                self.step(self.losses[k:k + 1])
            return self.losses
        if self._graph is None:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for k in range(iters):
                    self.step(self.losses[k:k + 1], stream=s)
            torch.cuda.current_stream().wait_stream(s)
            self._graph = g
        self._graph.replay()
        return self.losses
