"""GPU parity of the true knot gradients (NEXT-4) against the fp64 oracle
(oracle.surface_knot_grad / curve_knot_grad, pinned by finite differences and the
shift / scale invariants in test_oracle_pins.py), through the C ABI. Tolerance: normwise
1e-4 per direction per surface (or for the batch sum with shared knots), like the other
gradients (R16). The control-point gradient of the same call equals nurbs_surface_bwd's bitwise.
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
from test_gpu_parity import BWD_TOL, T  # noqa: E402

KTOL = BWD_TOL


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2104_14547_b200.build import build
    build()
    oracle.build()


def kerr(gpu, ref):
    gpu, ref = np.atleast_2d(gpu), np.atleast_2d(ref)
    sc = np.abs(ref).max(axis=1)
    sc[sc == 0] = 1.0
    return float(np.max(np.abs(gpu - ref).max(axis=1) / sc))


def run(w, g, tables=False):
    ctrl, U, V, u, v = T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v)
    tab = nb.Tables.build(nb.surface_shape(ctrl, U, u, v, w.p, w.q), U, V, u, v) if tables else None
    gc, gU, gV = nb.surface_bwd_knots(ctrl, U, V, u, v, T(g), w.p, w.q, tables=tab)
    plain = nb.surface_bwd(ctrl, U, V, u, v, T(g), w.p, w.q, tables=tab)
    torch.cuda.synchronize()
    assert torch.equal(gc, plain), "control gradient must equal nurbs_surface_bwd's bitwise"
    return gU.cpu().numpy(), gV.cpu().numpy()


def check(w, g=None, tables=False):
    g = w.grad_out() if g is None else g
    gU, gV = run(w, g, tables)
    rU, rV = oracle.surface_knot_grad(w.ctrl, w.U, w.V, w.u, w.v, g, w.p, w.q, w.knots_batched)
    if not w.knots_batched:
        rU, rV = rU[0], rV[0]
    assert kerr(gU, rU) <= KTOL and kerr(gV, rV) <= KTOL, (kerr(gU, rU), kerr(gV, rV))


@pytest.mark.parametrize("p,q", [(1, 1), (2, 3), (3, 3), (3, 1), (4, 2), (5, 5)])
@pytest.mark.parametrize("batched", [False, True])
def test_knot_grad_parity_degrees(p, q, batched):
    rng = np.random.default_rng(50 + 10 * p + q + (7 if batched else 0))
    n, m = int(rng.integers(p + 1, p + 8)), int(rng.integers(q + 1, q + 8))
    w = wl.surfaces(f"k{p}{q}", 3, n, m, p, q, 37, 29, seed=p + 5 * q, knots_batched=batched)
    check(w)


@pytest.mark.parametrize("B,p,q,n_v", [(16, 3, 3, 29), (40, 2, 5, 150), (23, 4, 1, 300)])
def test_knot_grad_shared_knots_batch_first_sum(B, p, q, n_v):
    """Shared knots with B >= 16: the assembly sums the per-surface weights over the batch
    first (two-level fixed tree) and differentiates once; against the oracle's batch sum."""
    w = wl.surfaces(f"kb{B}", B, 9, 11, p, q, 37, n_v, seed=B + p)
    check(w)


@pytest.mark.parametrize("p,q", [(1, 1), (3, 3), (5, 5), (2, 4)])
@pytest.mark.parametrize("B,batched", [(3, False), (3, True), (20, False)])
def test_knot_grad_span_moments(p, q, B, batched):
    """Shapes with >= 16 sample rows per knot span take the span-moment path (grid mode 4 +
    the per-span collocation assembly, nurbs_knots.cu): 5 spans x 20 rows, against the oracle
    (shared knots with B >= 16 sum the span moments over the batch first)."""
    w = wl.surfaces(f"ks{p}{q}", B, p + 5, q + 6, p, q, 100, 45, seed=p + 3 * q + B, knots_batched=batched)
    check(w)


def test_knot_grad_span_moments_tiled():
    """Span moments with several row blocks and column blocks (partials summed per span
    before the assembly) and with the precomputed tables."""
    w = wl.surfaces("kst", 1, 40, 10, 3, 3, 629, 300, seed=21)   # 37 spans x 17 rows, NCB = 3
    check(w)
    check(w, tables=True)
    w2 = wl.surfaces("kst5", 2, 64, 12, 3, 3, 1024, 256, seed=22)  # 61 spans x 16.8 rows
    check(w2)


def test_knot_grad_tiled_and_tables():
    """Several row and column blocks (the reduce path, several partials per sample)."""
    w = wl.surfaces("tiled", 1, 12, 10, 3, 3, 50, 260, seed=8)   # NRB = 9 row blocks, NCB = 3
    check(w)
    w2 = wl.config2()
    check(w2, tables=True)


def test_knot_grad_config1_curve():
    c = wl.config1()
    g = c.grad_out()
    ctrl, U, u = T(c.ctrl), T(c.U), T(c.u)
    gc, gU = nb.curve_bwd_knots(ctrl, U, u, T(g), c.p)
    plain = nb.curve_bwd(ctrl, U, u, T(g), c.p)
    torch.cuda.synchronize()
    assert torch.equal(gc, plain)
    ref = oracle.curve_knot_grad(c.ctrl, c.U, c.u, g, c.p)[0]
    assert kerr(gU.cpu().numpy(), ref) <= KTOL


def test_knot_grad_repeatable_and_shift_invariant_full_cfg4():
    """Full config 4 (4096 surfaces, shared knots: one gradient summed over the batch): bitwise
    repeatable, and sum_k dL/dU_k = -sum g . S_u with S_u from the (separately pinned) GPU
    derivative kernel — a property that holds at any size."""
    w = wl.config4()
    g = w.grad_out()
    a = run(w, g)
    b = run(w, g)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    _, Su, Sv, _ = nb.surface_derivs(T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v), 3, 3, with_points=False,
                                     with_normals=False)
    gt = T(g).double()
    su = float((gt * Su.double()).sum())
    sv = float((gt * Sv.double()).sum())
    scale = float(np.abs(a[0]).sum() + abs(su))
    assert abs(float(a[0].astype(np.float64).sum()) + su) <= 1e-4 * scale
    assert abs(float(a[1].astype(np.float64).sum()) + sv) <= 1e-4 * float(np.abs(a[1]).sum() + abs(sv))


def test_knot_grad_full_cfg4_batched_sampled():
    """Config 4 with per-surface knots at full size: sampled surfaces against the oracle."""
    w = wl.config4(knots_batched=True)
    g = w.grad_out()
    gU, gV = run(w, g)
    for k in (0, 4095):
        sub = wl.Surfaces("s", 3, 3, w.ctrl[k:k + 1], w.U[k:k + 1], w.V[k:k + 1], w.u, w.v, True)
        rU, rV = oracle.surface_knot_grad(sub.ctrl, sub.U, sub.V, sub.u, sub.v, g[k:k + 1], 3, 3, True)
        assert kerr(gU[k:k + 1], rU) <= KTOL and kerr(gV[k:k + 1], rV) <= KTOL


@pytest.mark.parametrize("shared", [True, False])
def test_knot_grad_cuda_graph_capture(shared):
    """The knot-gradient call forks its column-direction assembly onto a helper stream and
    joins it before returning (nurbs_api.cu): under CUDA-graph capture on a side stream the
    replayed graph must reproduce the eager results bitwise, and the eager call on another
    stream must not race with it (the join orders the helper stream's work)."""
    w = wl.config4(B=32) if shared else wl.config4(B=20, knots_batched=True)
    g = w.grad_out(5)
    ctrl, U, V, u, v, gout = T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v), T(g)
    sh = nb.surface_shape(ctrl, U, u, v, w.p, w.q)
    ws_b = nb.knots_workspace_bytes(sh)
    ws = torch.empty(max(ws_b, 1), dtype=torch.uint8, device=ctrl.device)
    gc, gU, gV = torch.empty_like(ctrl), torch.empty_like(U), torch.empty_like(V)
    call = lambda st: nb.nurbs_surface_bwd_knots(sh, ctrl, U, V, u, v, None, gout, gc, gU, gV, ws, ws_b, st)  # noqa: E731
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    call(s)
    torch.cuda.synchronize()
    ref = (gc.clone(), gU.clone(), gV.clone())
    for t in (gc, gU, gV):
        t.fill_(7.0)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        call(s)
    for _ in range(3):
        for t in (gc, gU, gV):
            t.fill_(-3.0)
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(gc, ref[0]) and torch.equal(gU, ref[1]) and torch.equal(gV, ref[2])


@pytest.mark.parametrize("seed", range(8))
def test_knot_grad_span_moments_fuzz(seed):
    """Span-moment mode on random shapes with non-uniform shared knots (one interior knot
    doubled where there is room: an empty span whose moments are zero), degrees 1..5, small and
    batch-first (B >= 16) batches, against the oracle at the stated tolerance."""
    rng = np.random.default_rng(900 + seed)
    p, q = int(rng.integers(1, 6)), int(rng.integers(1, 6))
    n, m = p + int(rng.integers(2, 7)), q + int(rng.integers(2, 7))
    n_u, n_v = 16 * (n - p) + int(rng.integers(0, 41)), int(rng.integers(5, 140))
    B = int(rng.choice([2, 17]))
    w = wl.surfaces(f"ksf{seed}", B, n, m, p, q, n_u, n_v, seed=seed)
    U = wl.random_clamped_knots(rng, n, p)
    if n - p - 1 >= 2:
        k = p + 1 + int(rng.integers(0, n - p - 2))
        U[k + 1] = U[k]
    w = wl.Surfaces(w.name, p, q, w.ctrl, U.astype(np.float32), w.V, w.u, w.v, False)
    check(w)
