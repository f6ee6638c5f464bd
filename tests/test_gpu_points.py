"""GPU parity of the paired (scattered) parameter points path (NEXT-1) against the fp64
oracle (oracle.surface_fwd_points / surface_bwd_points, pinned in test_oracle_pins.py),
through the C ABI. Tolerances as test_gpu_parity.py (north_star, R16): forward normwise
1e-5 per surface, gradients normwise 1e-4 per tensor per surface, knot gradients exactly
zero, bitwise repeatability.
"""
import numpy as np
import pytest

import oracle
import workloads as wl

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_14547_b200 as nb  # noqa: E402
from paper_2104_14547_b200 import _abi  # noqa: E402
from test_gpu_parity import BWD_TOL, FWD_TOL, T, bwd_err, fwd_err  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2104_14547_b200.build import build
    build()
    oracle.build()


def run(w, g, grad_knots=True):
    ctrl, U, V, uv, gout = T(w.ctrl), T(w.U), T(w.V), T(w.uv), T(g)
    out = nb.surface_points_fwd(ctrl, U, V, uv, w.p, w.q)
    gU = torch.full_like(U, 3.0) if grad_knots else None
    gV = torch.full_like(V, -2.0) if grad_knots else None
    grad = nb.surface_points_bwd(ctrl, U, V, uv, gout, w.p, w.q, grad_U=gU, grad_V=gV)
    torch.cuda.synchronize()
    if grad_knots:
        assert torch.count_nonzero(gU).item() == 0 and torch.count_nonzero(gV).item() == 0
    return out.cpu().numpy(), grad.cpu().numpy()


def check(w, g=None):
    g = w.grad_out() if g is None else g
    out, grad = run(w, g)
    ref = oracle.surface_fwd_points(w.ctrl, w.U, w.V, w.uv, w.p, w.q, w.knots_batched)
    assert fwd_err(out, ref, w.ctrl) <= FWD_TOL
    gref = oracle.surface_bwd_points(w.ctrl, w.U, w.V, w.uv, g, w.p, w.q, w.knots_batched)
    assert bwd_err(grad, gref, w.ctrl) <= BWD_TOL
    return out, grad


@pytest.mark.parametrize("p,q", [(1, 1), (2, 3), (3, 3), (3, 2), (4, 5), (5, 4), (5, 5), (1, 5)])
@pytest.mark.parametrize("batched", [False, True])
def test_points_parity_degrees(p, q, batched):
    rng = np.random.default_rng(10 * p + q + (100 if batched else 0))
    n, m = int(rng.integers(p + 1, p + 12)), int(rng.integers(q + 1, q + 12))
    w = wl.paired(f"pq{p}{q}", 3, n, m, p, q, 1537, seed=p * 7 + q, knots_batched=batched)
    check(w)


@pytest.mark.parametrize("B,N", [(1, 20000), (8, 3001), (600, 500), (2, 1), (5, 33)])
def test_points_parity_chunking(B, N):
    """Multi-chunk (partials + fixed-order reduce), single-chunk (in-kernel epilogue), tiny."""
    w = wl.paired(f"ch{B}_{N}", B, 16, 16, 3, 3, N, seed=B + N)
    check(w)


def test_points_one_heavy_cell_and_cfg4_net():
    """All points of a surface in one knot cell (one group walks them all), and cfg4's net."""
    w = wl.paired("heavy", 4, 16, 16, 3, 3, 6000, seed=9)
    w.uv[:2] = (w.uv[:2] * np.float32(0.05)).astype(np.float32)   # cells (0,0)/(0,1)/(1,0)/(1,1)
    w.uv[2] = np.float32(0.5)                                       # one exact knot pair
    check(w)


def test_points_repeatable_bitwise():
    w = wl.paired("rep", 6, 16, 16, 3, 3, 9000, seed=5)
    a = run(w, w.grad_out(), grad_knots=False)
    b = run(w, w.grad_out(), grad_knots=False)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_points_grid_coordinates_match_grid_path():
    """Paired points at the grid coordinates give the grid kernel's results (two different
    kernels and decompositions: equal within fp32 rounding)."""
    g = wl.config2()
    uu, vv = np.meshgrid(g.u, g.v, indexing="ij")
    uv = np.stack([uu.ravel(), vv.ravel()], -1)[None].astype(np.float32)
    gout = g.grad_out()
    ctrl, U, V = T(g.ctrl), T(g.U), T(g.V)
    grid_out = nb.surface_fwd(ctrl, U, V, T(g.u), T(g.v), 3, 3).cpu().numpy()
    grid_grad = nb.surface_bwd(ctrl, U, V, T(g.u), T(g.v), T(gout), 3, 3).cpu().numpy()
    pts_out = nb.surface_points_fwd(ctrl, U, V, T(uv), 3, 3).cpu().numpy()
    pts_grad = nb.surface_points_bwd(ctrl, U, V, T(uv), T(gout.reshape(1, -1, 3)), 3, 3).cpu().numpy()
    assert fwd_err(pts_out, grid_out.reshape(1, -1, 3), g.ctrl) <= FWD_TOL
    assert bwd_err(pts_grad, grid_grad.astype(np.float64), g.ctrl) <= BWD_TOL


def test_points_empty_and_errors():
    w = wl.paired("empty", 2, 8, 8, 3, 3, 0, seed=1)
    ctrl, U, V = T(w.ctrl), T(w.U), T(w.V)
    uv = torch.zeros((2, 0, 2), device=ctrl.device)
    out = nb.surface_points_fwd(ctrl, U, V, uv, 3, 3)
    assert out.shape == (2, 0, 3)
    grad = nb.surface_points_bwd(ctrl, U, V, uv, torch.zeros((2, 0, 3), device=ctrl.device), 3, 3)
    assert torch.count_nonzero(grad).item() == 0
    # n_v must be 1
    sh = nb.points_shape(ctrl, U, uv, 3, 3)
    sh.n_v = 2
    with pytest.raises(_abi.NurbsError) as e:
        nb.nurbs_surface_points_fwd(sh, ctrl, U, V, uv, out)
    assert e.value.status == 1
    # a net too large for the in-smem reduction is refused, not mis-computed
    big = wl.paired("big", 1, 64, 64, 3, 3, 10, seed=2)
    with pytest.raises(_abi.NurbsError) as e:
        nb.surface_points_bwd(T(big.ctrl), T(big.U), T(big.V), T(big.uv), T(big.grad_out()), 3, 3)
    assert e.value.status == 2
    # checked mode: a point outside the domain
    w2 = wl.paired("bad", 2, 8, 8, 3, 3, 50, seed=3)
    w2.uv[1, 17, 1] = 1.25
    sh2 = nb.points_shape(T(w2.ctrl), T(w2.U), T(w2.uv), 3, 3)
    with pytest.raises(_abi.NurbsError) as e:
        nb.nurbs_validate_points(sh2, T(w2.ctrl), T(w2.U), T(w2.V), T(w2.uv))
    assert e.value.status == 4 and "v of a point" in str(e.value)
    nb.nurbs_validate_points(sh2, T(w.ctrl), T(w.U), T(w.V), T(wl.paired("ok", 2, 8, 8, 3, 3, 50, seed=3).uv))


def test_points_full_size_sampled():
    """cfg4p (4096 x 16x16 bicubic, 16384 scattered points each) in the launch configuration
    bench.py times; surfaces are independent, so sampled surfaces are checked exactly."""
    w = wl.config4_paired()
    g = w.grad_out()
    out, grad = run(w, g)
    for k in (0, 1, 2047, 4095):
        sub = wl.PairedSurfaces("s", 3, 3, w.ctrl[k:k + 1], w.U, w.V, w.uv[k:k + 1])
        ref = oracle.surface_fwd_points(sub.ctrl, sub.U, sub.V, sub.uv, 3, 3)
        assert fwd_err(out[k:k + 1], ref, sub.ctrl) <= FWD_TOL
        gref = oracle.surface_bwd_points(sub.ctrl, sub.U, sub.V, sub.uv, g[k:k + 1], 3, 3)
        assert bwd_err(grad[k:k + 1], gref, sub.ctrl) <= BWD_TOL
    assert np.isfinite(out).all() and np.isfinite(grad).all()
