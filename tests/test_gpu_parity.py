"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle on the same
seeded fp32 inputs. Tolerances (north_star, normwise per reading R16 of DESIGN.md §3):
  spans / indices      bit-exact
  forward              max|S_gpu - S_ref| / max|P|          <= 1e-5  per surface
  gradients            max|d_gpu - d_ref| / max|d_ref|      <= 1e-4  per tensor (dP, dw) per surface
  knot gradients       exactly zero
  repeatability        bitwise
"""
import ctypes
import os

import numpy as np
import pytest

import oracle
import workloads as wl
from conftest import record

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_14547_b200 as nb  # noqa: E402
from paper_2104_14547_b200 import _abi  # noqa: E402

DEV = torch.device("cuda:0")
FWD_TOL, BWD_TOL = 1e-5, 1e-4


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2104_14547_b200.build import build
    build()
    oracle.build()


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def fwd_err(gpu, ref, ctrl, name=None):
    """per-surface normwise forward error: max|S_gpu - S_ref| / max|P| (R16)"""
    B = ctrl.shape[0]
    e = np.abs(gpu.reshape(B, -1) - ref.reshape(B, -1)).max(axis=1)
    scale = np.abs(ctrl[..., :3].reshape(B, -1)).max(axis=1)
    err = float(np.max(e / scale))
    record(name, "fwd", err)
    return err


def bwd_err_parts(gpu, ref, ctrl=None):
    """(dP error, dw error): per surface max|d_gpu - d_ref| / max|d_ref| for each tensor (R16),
    worst over the surfaces. The scale is the ORACLE's max|d_ref| (never the GPU's).

    One exception, for dw only: when max|dw_ref| < 1e-6 max_ij |P_ij||dQ_xyz,ij| (dQ_xyz = dP/w),
    dw = P.dQ_xyz + dQ_w is an exact cancellation of two terms (e.g. a single sample at a clamped
    corner, where S = P_00 and Eq.9's (P - S) factor is 0). There the reference is pure rounding
    noise (~1e-16) and the scale is the size of the cancelling term, max_ij |P_ij||dQ_xyz,ij|
    (R16). No workload with a non-degenerate dw takes this branch."""
    B = ref.shape[0]
    g = np.asarray(gpu, dtype=np.float64).reshape(B, -1, 4)
    r = np.asarray(ref, dtype=np.float64).reshape(B, -1, 4)
    eP = np.abs(g[..., :3] - r[..., :3]).reshape(B, -1).max(axis=1)
    sP = np.abs(r[..., :3]).reshape(B, -1).max(axis=1)
    ew = np.abs(g[..., 3] - r[..., 3]).max(axis=1)
    sw = np.abs(r[..., 3]).max(axis=1)
    if ctrl is not None:
        c = np.asarray(ctrl, dtype=np.float64).reshape(B, -1, 4)
        first = (np.abs(c[..., :3]) * np.abs(r[..., :3])).sum(axis=2) / c[..., 3]  # sum |P||dQ_xyz|, dQ = dP/w
        first = first.max(axis=1)
        sw = np.where(sw < 1e-6 * first, first, sw)
    sP[sP == 0] = 1.0
    sw[sw == 0] = 1.0
    return float(np.max(eP / sP)), float(np.max(ew / sw))


def bwd_err(gpu, ref, ctrl=None, name=None):
    """max of the dP and dw errors of bwd_err_parts (each must meet BWD_TOL = 1e-4)"""
    eP, ew = bwd_err_parts(gpu, ref, ctrl)
    record(name, "dP", eP)
    record(name, "dw", ew)
    return max(eP, ew)


def run_surface(w, g, tables=False, grad_knots=True):
    ctrl, U, V, u, v, gout = T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v), T(g)
    tab = None
    if tables:
        sh = nb.surface_shape(ctrl, U, u, v, w.p, w.q)
        tab = nb.Tables.build(sh, U, V, u, v)
    out = nb.surface_fwd(ctrl, U, V, u, v, w.p, w.q, tables=tab)
    gU = torch.full_like(U, 3.0) if grad_knots else None
    gV = torch.full_like(V, -2.0) if grad_knots else None
    grad = nb.surface_bwd(ctrl, U, V, u, v, gout, w.p, w.q, tables=tab, grad_U=gU, grad_V=gV)
    torch.cuda.synchronize()
    if grad_knots:
        assert torch.all(gU == 0) and torch.all(gV == 0)
    return out.cpu().numpy(), grad.cpu().numpy()


def check_surface(w, gseed=0, tables=False, fwd_tol=FWD_TOL, bwd_tol=BWD_TOL):
    g = w.grad_out(gseed)
    out, grad = run_surface(w, g, tables)
    ref_out = oracle.surface_fwd(w.ctrl, w.U, w.V, w.u, w.v, w.p, w.q, w.knots_batched)
    ref_grad = oracle.surface_bwd(w.ctrl, w.U, w.V, w.u, w.v, g, w.p, w.q, w.knots_batched)
    ef, eb = fwd_err(out, ref_out, w.ctrl, w.name), bwd_err(grad, ref_grad, w.ctrl, w.name)
    assert ef <= fwd_tol, f"{w.name}: forward error {ef:.3e}"
    assert eb <= bwd_tol, f"{w.name}: backward error {eb:.3e}"
    return ef, eb


# --------------------------------------------------------------------------- configs
def test_config1_curve_and_fd():
    c = wl.config1()
    g = c.grad_out()
    ctrl, U, u, gout = T(c.ctrl), T(c.U), T(c.u), T(g)
    gU = torch.full_like(U, 1.0)
    out = nb.curve_fwd(ctrl, U, u, c.p).cpu().numpy()
    grad = nb.curve_bwd(ctrl, U, u, gout, c.p, grad_U=gU).cpu().numpy()
    assert torch.all(gU == 0)
    ref = oracle.curve_fwd(c.ctrl, c.U, c.u, c.p)
    refg = oracle.curve_bwd(c.ctrl, c.U, c.u, g, c.p)
    assert fwd_err(out, ref, c.ctrl) <= FWD_TOL
    assert bwd_err(grad, refg) <= BWD_TOL
    # config 1 asks for fwd+bwd vs finite differences: central FD of the fp64 oracle
    fd = np.zeros_like(refg)
    h = 1e-6
    base = c.ctrl.astype(np.float64)
    for idx in np.ndindex(base.shape):
        cp, cm = base.copy(), base.copy()
        cp[idx] += h
        cm[idx] -= h
        fd[idx] = (np.sum(oracle.curve_fwd(cp, c.U, c.u, c.p) * g) - np.sum(oracle.curve_fwd(cm, c.U, c.u, c.p) * g)) / (2 * h)
    assert bwd_err(grad, fd) <= BWD_TOL


@pytest.mark.parametrize("tables", [False, True])
def test_config2(tables):
    check_surface(wl.config2(), tables=tables)


def test_config3():
    check_surface(wl.config3())


def test_config4_small_batch():
    check_surface(wl.config4(B=48))


def test_config4_batched_knots():
    check_surface(wl.config4(B=24, knots_batched=True))


def test_config5_shape_reduced_grid():
    """256x256 net on a 1024x1024 grid: many row blocks and column blocks -> workspace + reduce."""
    w = wl.config5(n_u=1024, n_v=1024)
    sh = _abi.nurbs_shape(1, 256, 256, 3, 3, 1024, 1024, 0)
    assert nb.bwd_workspace_bytes(sh) > 0
    check_surface(w)


# --------------------------------------------------------------------------- degrees / shapes
@pytest.mark.parametrize("p,q", [(1, 1), (1, 5), (2, 3), (3, 2), (4, 4), (5, 1), (5, 5)])
def test_degrees(p, q):
    rng_seed = 10 * p + q
    w = wl.surfaces(f"deg{p}{q}", B=3, n=p + 9, m=q + 6, p=p, q=q, n_u=70, n_v=131, seed=rng_seed, knots_batched=(p % 2 == 1))
    check_surface(w, tables=False)


@pytest.mark.parametrize("n_v", [1, 3, 130, 257, 300])
def test_ragged_columns_and_non_tma_path(n_v):
    """n_v not a multiple of 4 takes the non-TMA path; n_v > 128 has ragged column blocks."""
    w = wl.surfaces("ragged", B=2, n=11, m=9, p=3, q=3, n_u=45, n_v=n_v, seed=n_v)
    check_surface(w)


@pytest.mark.parametrize("n_u,n_v,tables", [(45, 64, False), (13, 196, True), (70, 132, False), (9, 256, False),
                                             (37, 324, True), (200, 68, True)])
def test_tensor_map_path(n_u, n_v, tables):
    """n_v % 4 == 0 and rows not contiguous per stage: the 2-D TMA tensor path (two 64-column
    boxes per 8-row stage, per-row fallback for a partial last stage, ragged second box; with
    tables the forward's cp.async row-table prefetch over several 64-row chunks). Against the
    oracle, and bitwise against the per-thread (non-TMA) path."""
    w = wl.surfaces("tmap", B=2, n=11, m=9, p=3, q=3, n_u=n_u, n_v=n_v, seed=n_u + n_v)
    check_surface(w, tables=tables)
    g = w.grad_out(2)
    a = run_surface(w, g, tables)
    with nb.path_flags(no_tma=True):
        b = run_surface(w, g, tables)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


@pytest.mark.parametrize("force_no_tma", [False, True])
def test_tma_and_direct_paths_agree(force_no_tma):
    w = wl.config4(B=8)
    g = w.grad_out(1)
    a = run_surface(w, g)
    with nb.path_flags(no_tma=force_no_tma):
        b = run_surface(w, g)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


@pytest.mark.parametrize("case", ["cfg2", "cfg4", "m32", "tiled", "ragged", "tmap_tail"])
def test_tensor_core_backward_matches_simt_and_oracle(case):
    """The tcgen05 backward (3xTF32 MMAs, nurbs_bwd_tc.cu; NURBS_PATH_TC) covers p = q = 3 and
    m <= 32; the SIMT grid kernel (the default) is an independent GPU implementation of the same
    transposed banded product. Both against the oracle at the stated tolerance, against each
    other within rounding, and the tensor-core path bitwise repeatable, TMA or not."""
    w = {"cfg2": lambda: wl.config2(),
         "cfg4": lambda: wl.config4(B=32),
         "m32": lambda: wl.surfaces("m32", B=3, n=20, m=32, p=3, q=3, n_u=150, n_v=256, seed=12),
         "tiled": lambda: wl.surfaces("tl", B=2, n=120, m=24, p=3, q=3, n_u=1500, n_v=300, seed=13),
         "ragged": lambda: wl.surfaces("rg", B=2, n=14, m=11, p=3, q=3, n_u=77, n_v=333, seed=14),
         "tmap_tail": lambda: wl.surfaces("tt", B=2, n=30, m=9, p=3, q=3, n_u=203, n_v=196, seed=15)}[case]()
    g = w.grad_out(7)
    ref = oracle.surface_bwd(w.ctrl, w.U, w.V, w.u, w.v, g, w.p, w.q)
    with nb.path_flags(tc=True):
        tc1 = run_surface(w, g)[1]
        tc2 = run_surface(w, g)[1]
    with nb.path_flags(tc=True, no_tma=True):
        tc3 = run_surface(w, g)[1]
    np.testing.assert_array_equal(tc1, tc2)
    np.testing.assert_array_equal(tc1, tc3)
    simt = run_surface(w, g)[1]
    assert bwd_err(tc1, ref, w.ctrl, f"tc-{case}") <= BWD_TOL
    assert bwd_err(simt, ref, w.ctrl, f"simt-{case}") <= BWD_TOL
    assert bwd_err(tc1, simt.astype(np.float64), w.ctrl) <= BWD_TOL


def test_sparse_samples_dense_knots():
    """Fewer samples than spans: the row window jumps by more than p+1 rows."""
    w = wl.surfaces("sparse", B=2, n=60, m=40, p=3, q=2, n_u=7, n_v=5, seed=3)
    check_surface(w)


# --------------------------------------------------------------------------- adversarial
def adversarial_surface(seed, p=3, q=3, n=12, m=10, mult=None, wlo=0.05, whi=20.0):
    rng = np.random.default_rng(seed)
    def knots(n, p):
        inner = np.sort(rng.uniform(0.05, 0.95, n - p - 1)).astype(np.float32)
        if mult and len(inner) > mult:
            inner[1:1 + mult] = inner[1]          # an interior knot of multiplicity `mult`
        return np.concatenate([np.zeros(p + 1, np.float32), np.sort(inner), np.ones(p + 1, np.float32)])
    U, V = knots(n, p), knots(m, q)
    # samples: every knot, its fp32 neighbours, 0 and 1, plus random
    def samples(K):
        s = set(K.tolist())
        for k in K:
            s.add(float(np.nextafter(np.float32(k), np.float32(2))))
            s.add(float(np.nextafter(np.float32(k), np.float32(-1))))
        s |= set(rng.uniform(0, 1, 40).astype(np.float32).tolist())
        return np.array(sorted(x for x in s if 0.0 <= x <= 1.0), dtype=np.float32)
    ctrl = wl.random_net(rng, (2, n, m), wlo, whi)
    return wl.Surfaces("adv", p, q, ctrl, U, V, samples(U), samples(V))


@pytest.mark.parametrize("seed,mult", [(0, None), (1, 2), (2, 3)])
def test_adversarial_knots_and_weights(seed, mult):
    w = adversarial_surface(seed, mult=mult)
    check_surface(w, tables=bool(seed % 2))


def test_spans_bit_exact_in_tables():
    for w in [wl.config2(), wl.config3(), adversarial_surface(5, mult=3), wl.config5(n_u=8192, n_v=64)]:
        sh = _abi.nurbs_shape(w.B, w.n, w.m, w.p, w.q, w.n_u, w.n_v, 0)
        U, V, u, v = T(w.U), T(w.V), T(w.u), T(w.v)
        tab = nb.Tables.build(sh, U, V, u, v)
        torch.cuda.synchronize()
        buf = tab.buf.cpu().numpy()
        hdr = buf[:64].view(np.int32)
        assert hdr[0] == 0x4E524253
        np_r = hdr[5]
        off = 256
        span_u = buf[off:off + 4 * w.n_u].view(np.int32)
        su, Nu = oracle.spans(w.n, w.p, w.U, w.u)
        np.testing.assert_array_equal(span_u, su)
        off = (off + 4 * w.n_u + 255) // 256 * 256
        Nu_gpu = buf[off:off + 4 * w.n_u * np_r].view(np.float32).reshape(w.n_u, np_r)[:, :w.p + 1]
        assert np.max(np.abs(Nu_gpu - Nu)) <= 2e-6
        off = (off + 4 * w.n_u * np_r + 255) // 256 * 256
        sv, _ = oracle.spans(w.m, w.q, w.V, w.v)
        np.testing.assert_array_equal(buf[off:off + 4 * w.n_v].view(np.int32), sv)


def test_config1_hits_interior_knots_exactly():
    c = wl.config1()
    sh = _abi.nurbs_shape(1, c.n, 1, c.p, 0, c.n_u, 1, 0)
    tab = nb.Tables.build(sh, T(c.U), None, T(c.u), None)
    torch.cuda.synchronize()
    buf = tab.buf.cpu().numpy()
    hdr = buf[:64].view(np.int32)
    # curve tables: the row part is empty, the columns are the curve (header is 256 bytes)
    off = 256
    span = buf[off:off + 4 * c.n_u].view(np.int32)
    su, _ = oracle.spans(c.n, c.p, c.U, c.u)
    np.testing.assert_array_equal(span, su)
    assert span[33] == 4 and span[66] == 5 and hdr[8] == c.n_u


# --------------------------------------------------------------------------- exactness pins on GPU
def test_quarter_circle_radius_fp32():
    s2 = np.float32(np.sqrt(2.0) / 2.0)
    ctrl = np.array([[[1, 0, 0, 1], [1, 1, 0, s2], [0, 1, 0, 1]]], dtype=np.float32)
    U = np.array([0, 0, 0, 1, 1, 1], dtype=np.float32)
    u = wl.uniform_grid(1000)
    out = nb.curve_fwd(T(ctrl), T(U), T(u), 2).cpu().numpy()
    r = np.hypot(out[0, :, 0].astype(np.float64), out[0, :, 1].astype(np.float64))
    assert np.max(np.abs(r - 1.0)) <= 1e-6


def test_determinism_bitwise():
    for w in [wl.config4(B=16), wl.config5(n_u=512, n_v=512)]:
        g = w.grad_out(3)
        a = run_surface(w, g)
        b = run_surface(w, g)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])


# --------------------------------------------------------------------------- edge cases
def test_empty_inputs():
    w = wl.surfaces("e", B=2, n=6, m=6, p=3, q=3, n_u=5, n_v=5, seed=1)
    ctrl, U, V = T(w.ctrl), T(w.U), T(w.V)
    u0 = torch.empty(0, device=DEV)
    v = T(w.v)
    out = nb.surface_fwd(ctrl, U, V, u0, v, 3, 3)
    assert out.shape == (2, 0, 5, 3)
    grad = nb.surface_bwd(ctrl, U, V, u0, v, torch.empty(2, 0, 5, 3, device=DEV), 3, 3,
                          grad_ctrl=torch.full_like(ctrl, 5.0))
    torch.cuda.synchronize()
    assert torch.all(grad == 0)
    out = nb.surface_fwd(ctrl[:0], U, V, T(w.u), v, 3, 3)
    assert out.shape[0] == 0


def test_single_sample_and_corner_interpolation():
    w = wl.surfaces("one", B=3, n=5, m=7, p=2, q=3, n_u=1, n_v=1, seed=2)
    out, grad = run_surface(w, w.grad_out(0))
    np.testing.assert_allclose(out[:, 0, 0], w.ctrl[:, 0, 0, :3], rtol=0, atol=1e-6)   # S(0,0) = P_00
    check_surface(w)


def test_errors_and_checked_mode():
    w = wl.surfaces("err", B=1, n=8, m=8, p=3, q=3, n_u=16, n_v=16, seed=4)
    ctrl, U, V, u, v = T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v)
    sh = nb.surface_shape(ctrl, U, u, v, 3, 3)
    nb.nurbs_validate(sh, ctrl, U, V, u, v)
    bad = U.clone(); bad[5], bad[6] = 0.9, 0.1
    with pytest.raises(nb.NurbsError) as e:
        nb.nurbs_validate(sh, ctrl, bad, V, u, v)
    assert e.value.status == 3
    with pytest.raises(nb.NurbsError) as e:
        nb.nurbs_validate(sh, ctrl, U, V, u.flip(0).contiguous(), v)
    assert e.value.status == 6
    with pytest.raises(nb.NurbsError) as e:
        nb.nurbs_validate(sh, ctrl, U, V, u - 0.5, v)
    assert e.value.status in (4, 6)
    neg = ctrl.clone(); neg[0, 2, 3, 3] = -1.0
    with pytest.raises(nb.NurbsError) as e:
        nb.nurbs_validate(sh, neg, U, V, u, v)
    assert e.value.status == 5
    with pytest.raises(nb.NurbsError) as e:
        nb.Tables.build(sh, bad, V, u, v)
    assert e.value.status == 3
    big = wl.config5(n_u=256, n_v=256)
    c5 = T(big.ctrl)
    sh5 = nb.surface_shape(c5, T(big.U), T(big.u), T(big.v), 3, 3)
    ws = nb.bwd_workspace_bytes(sh5)
    with pytest.raises(nb.NurbsError) as e:
        nb.nurbs_surface_bwd(sh5, c5, T(big.U), T(big.V), T(big.u), T(big.v), None,
                             torch.zeros(1, 256, 256, 3, device=DEV), torch.empty_like(c5), None, None,
                             torch.empty(16, dtype=torch.uint8, device=DEV), 16)
    assert e.value.status == 8 and ws > 16


@pytest.mark.parametrize("case", ["cfg4", "tiled", "tmap", "curve"])
def test_unsorted_samples_unchecked_stay_in_bounds(case):
    """Unchecked mode with reversed / shuffled u and v (invalid input: the grid must be sorted,
    include/nurbs.h). Values are unspecified, but every call must complete without a CUDA
    fault (run this file under compute-sanitizer memcheck to see out-of-bounds accesses:
    scripts/gpu_sanitize.sh)."""
    rng = np.random.default_rng(11)
    if case == "curve":
        c = wl.config1()
        u = c.u[rng.permutation(len(c.u))].copy()
        out = nb.curve_fwd(T(c.ctrl), T(c.U), T(u), c.p)
        nb.curve_bwd(T(c.ctrl), T(c.U), T(u), torch.ones_like(out), c.p)
        torch.cuda.synchronize()
        return
    w = {"cfg4": lambda: wl.config4(B=8), "tiled": lambda: wl.config5(n_u=700, n_v=520),
         "tmap": lambda: wl.surfaces("um", B=2, n=11, m=9, p=3, q=3, n_u=45, n_v=200, seed=9)}[case]()
    for u, v in [(w.u[::-1].copy(), w.v[::-1].copy()), (w.u[rng.permutation(w.n_u)].copy(), w.v[rng.permutation(w.n_v)].copy()),
                 (w.u, w.v[::-1].copy()), (w.u[::-1].copy(), w.v)]:
        out = nb.surface_fwd(T(w.ctrl), T(w.U), T(w.V), T(u), T(v), w.p, w.q)
        g = torch.ones_like(out)
        nb.surface_bwd(T(w.ctrl), T(w.U), T(w.V), T(u), T(v), g, w.p, w.q)
        torch.cuda.synchronize()


# --------------------------------------------------------------------------- full BASELINE sizes
def check_invariants(grad, g, out, ctrl, tol=1e-5, name=None):
    """Exact identities of Eq.8/9 at every surface, any size:
         sum_ij dP_ij = sum_pts g            (translation)
         sum_ij w_ij dw_ij = 0               (S is homogeneous of degree 0 in w)
         sum_ij P_ij . dP_ij = sum_pts g . S (S is linear in P)
    Scale: max|P| * sum_pts |g| per surface, which bounds every term (|S| <= max|P|: convex
    hull, w > 0) and comes from neither the oracle nor the GPU gradient."""
    B = ctrl.shape[0]
    c = np.asarray(ctrl, dtype=np.float64).reshape(B, -1, 4)
    d = np.asarray(grad, dtype=np.float64).reshape(B, -1, 4)
    g64 = np.asarray(g, dtype=np.float64).reshape(B, -1, 3)
    S = np.asarray(out, dtype=np.float64).reshape(B, -1, 3)
    scale = np.abs(c[..., :3]).max(axis=(1, 2)) * np.abs(g64).sum(axis=(1, 2))
    scale[scale == 0] = 1.0
    e_t = np.abs(d[..., :3].sum(axis=1) - g64.sum(axis=1)).max(axis=1) / (np.abs(g64).sum(axis=(1, 2)) + 1e-300)
    e_w = np.abs((c[..., 3] * d[..., 3]).sum(axis=1)) / scale
    e_p = np.abs((c[..., :3] * d[..., :3]).sum(axis=(1, 2)) - (g64 * S).sum(axis=(1, 2))) / scale
    worst = float(max(e_t.max(), e_w.max(), e_p.max()))
    record(name, "invariants", worst)
    assert e_t.max() <= tol, f"translation invariant {e_t.max():.3e}"
    assert e_w.max() <= tol, f"weight-scale invariant {e_w.max():.3e}"
    assert e_p.max() <= tol, f"linearity invariant {e_p.max():.3e}"


def test_config4_full_size():
    """The bench workload (B=4096, 16x16, 128^2) in the bench launch configuration, EVERY
    surface against the fp64 oracle (threads over chunks of surfaces), plus the three exact
    gradient invariants at every surface."""
    w = wl.config4()
    g = w.grad_out(4)
    out, grad = run_surface(w, g, tables=True)
    chunks = [(k, min(k + 128, w.B)) for k in range(0, w.B, 128)]

    def job(k0, k1):
        c = w.ctrl[k0:k1]
        ro = oracle.surface_fwd(c, w.U, w.V, w.u, w.v, w.p, w.q)
        rg = oracle.surface_bwd(c, w.U, w.V, w.u, w.v, g[k0:k1], w.p, w.q)
        return fwd_err(out[k0:k1], ro, c), bwd_err_parts(grad[k0:k1], rg, c)

    res = oracle.pmap(job, chunks)
    ef = max(r[0] for r in res)
    eP = max(r[1][0] for r in res)
    ew = max(r[1][1] for r in res)
    record("cfg4 full", "fwd", ef); record("cfg4 full", "dP", eP); record("cfg4 full", "dw", ew)
    assert ef <= FWD_TOL, f"forward {ef:.3e}"
    assert eP <= BWD_TOL and ew <= BWD_TOL, f"dP {eP:.3e} dw {ew:.3e}"
    check_invariants(grad, g, out, w.ctrl, name="cfg4 full")


def test_config5_full_size():
    """One 256x256 net on the 8192^2 grid in the bench launch configuration: the whole output
    and the whole gradient against the fp64 oracle. The oracle runs on blocks of u-rows in
    threads; the per-block gradients (Eq.8/9 sums over the block's points) are added in block
    order in fp64 (SURVEY.md §8(c) Threading)."""
    w = wl.config5()
    g = w.grad_out(5)
    out, grad = run_surface(w, g, tables=True)
    rb = 256
    blocks = [(a, min(a + rb, w.n_u)) for a in range(0, w.n_u, rb)]

    def job(a0, a1):
        ro = oracle.surface_fwd(w.ctrl, w.U, w.V, w.u[a0:a1], w.v, w.p, w.q)
        e = float(np.abs(out[:, a0:a1] - ro).max())
        rg = oracle.surface_bwd(w.ctrl, w.U, w.V, w.u[a0:a1], w.v, g[:, a0:a1], w.p, w.q)
        return e, rg

    res = oracle.pmap(job, blocks)
    ef = max(r[0] for r in res) / float(np.abs(w.ctrl[..., :3]).max())
    ref = np.zeros_like(res[0][1])
    for r in res:
        ref += r[1]
    eP, ew = bwd_err_parts(grad, ref, w.ctrl)
    record("cfg5 full", "fwd", ef); record("cfg5 full", "dP", eP); record("cfg5 full", "dw", ew)
    assert ef <= FWD_TOL, f"forward {ef:.3e}"
    assert eP <= BWD_TOL and ew <= BWD_TOL, f"dP {eP:.3e} dw {ew:.3e}"
    check_invariants(grad, g, out, w.ctrl, name="cfg5 full")


# --------------------------------------------------------------------------- per-rank shard shapes
@pytest.mark.parametrize("B", [512, 100, 128, 127, 3])
def test_config4_rank_shard_plans(B):
    """Config 4's per-rank batch at G = 8 (B = 512: one tile per surface), the direct/tiled
    switch of the plan (B = 128 direct, 127 tiled + cross-tile reduce) and small batches, in the
    bench launch configuration (tables), against the fp64 oracle (every surface up to 128, 32
    sampled for B = 512); the gradient is bitwise repeatable."""
    w = wl.config4(B=B)
    g = w.grad_out(11)
    pl = nb.grid_plan(nb.nurbs_shape(B, 16, 16, 3, 3, 128, 128, 0))
    assert pl["direct"] == (1 if B >= 128 else 0)
    out, grad = run_surface(w, g, tables=True)
    np.testing.assert_array_equal(grad, run_surface(w, g, tables=True)[1])
    idx = np.arange(B) if B <= 128 else np.random.default_rng(3).choice(B, 32, replace=False)
    c = w.ctrl[idx]
    ro = oracle.surface_fwd(c, w.U, w.V, w.u, w.v, w.p, w.q)
    rg = oracle.surface_bwd(c, w.U, w.V, w.u, w.v, g[idx], w.p, w.q)
    ef, eb = fwd_err(out[idx], ro, c, f"cfg4 B={B}"), bwd_err(grad[idx], rg, c, f"cfg4 B={B}")
    assert ef <= FWD_TOL and eb <= BWD_TOL, (ef, eb)


def test_config5_row_window_shards():
    """Config 5's point sharding as bench.py runs it at G = 8: each rank's u-slab evaluated on
    its sub-net (dist.row_window). The forward equals the full-net forward of the same rows
    BITWISE (same spans, same knots, same operations); the windowed partial gradients, placed
    at their row offsets and summed, match the fp64 oracle's unsharded gradient."""
    from paper_2104_14547_b200 import dist as nbd
    w = wl.config5(n_u=2048, n_v=1024)
    g = w.grad_out(12)
    ctrl, U, V, u, v = T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v)
    full_out = nb.surface_fwd(ctrl, U, V, u, v, w.p, w.q).cpu().numpy()
    total = np.zeros((1, w.n, w.m, 4), dtype=np.float64)
    G = 8
    for r in range(G):
        a0, a1 = nbd.shard_range(w.n_u, G, r)
        r0, r1 = nbd.row_window(w.U, w.p, w.n, float(w.u[a0]), float(w.u[a1 - 1]))
        assert r1 - r0 < w.n
        sc, sU, su = T(w.ctrl[:, r0:r1]), T(w.U[r0:r1 + w.p + 1]), T(w.u[a0:a1])
        sh = nb.surface_shape(sc, sU, su, v, w.p, w.q)
        tab = nb.Tables.build(sh, sU, V, su, v)
        o = nb.surface_fwd(sc, sU, V, su, v, w.p, w.q, tables=tab).cpu().numpy()
        assert np.array_equal(o, full_out[:, a0:a1]), f"rank {r}: windowed forward differs"
        gr = nb.surface_bwd(sc, sU, V, su, v, T(g[:, a0:a1]), w.p, w.q, tables=tab).cpu().numpy()
        total[:, r0:r1] += gr
    blocks = [(a, min(a + 256, w.n_u)) for a in range(0, w.n_u, 256)]
    parts = oracle.pmap(lambda a0, a1: oracle.surface_bwd(w.ctrl, w.U, w.V, w.u[a0:a1], w.v, g[:, a0:a1], w.p, w.q),
                        blocks)
    ref = np.sum(parts, axis=0)
    eP, ew = bwd_err_parts(total, ref, w.ctrl)
    record("cfg5 windows G=8", "dP", eP); record("cfg5 windows G=8", "dw", ew)
    assert eP <= BWD_TOL and ew <= BWD_TOL, (eP, ew)


# --------------------------------------------------------------------------- fused fitting step (NEXT-2)
def oracle_fit(ctrl0, w, T, lr, iters):
    """fp64 oracle loop of the fitting step: L = mean |S - T|^2, SGD on P and w (Eq.14)."""
    c = ctrl0.astype(np.float64).copy()
    N = T.shape[1] * T.shape[2] * T.shape[0]
    losses, grads = [], []
    for _ in range(iters):
        S = oracle.surface_fwd(c, w.U, w.V, w.u, w.v, w.p, w.q)
        d = S - T
        losses.append(np.sum(d * d) / N)
        g = oracle.surface_bwd(c, w.U, w.V, w.u, w.v, 2.0 * d / N, w.p, w.q)
        grads.append(g)
        c = c - lr * g
    return np.array(losses), grads, c


@pytest.mark.parametrize("n_s,iters", [(128, 60), (512, 100)])  # config 3: first 100 iterations
def test_fit_step_trajectory(n_s, iters):
    truth, init = wl.config3_fit(n_s=n_s)
    T64 = oracle.surface_fwd(truth.ctrl, truth.U, truth.V, truth.u, truth.v, 3, 3)
    Tf = T64.astype(np.float32)
    lr = 200.0
    ref_loss, ref_grads, ref_ctrl = oracle_fit(init.ctrl, init, Tf.astype(np.float64), lr, iters)
    ctrl = T(init.ctrl)
    fitter = nb.SurfaceFitter(ctrl, T(init.U), T(init.V), T(init.u), T(init.v), T(Tf), 3, 3, lr)
    # one un-graphed step first: loss, gradient and update at iteration 0
    loss0 = torch.zeros(1, device=DEV)
    fitter.step(loss0)
    torch.cuda.synchronize()
    assert abs(loss0.item() - ref_loss[0]) <= 1e-5 * ref_loss[0]
    assert bwd_err(fitter.grad.cpu().numpy(), ref_grads[0], init.ctrl) <= BWD_TOL
    # the remaining iterations in one CUDA graph
    hist = fitter.run(iters - 1).cpu().numpy()
    losses = np.concatenate([[loss0.item()], hist])
    assert np.max(np.abs(losses - ref_loss)) / np.max(ref_loss) <= 1e-4
    assert ref_loss[-1] < 0.5 * ref_loss[0]                   # it actually fits
    got = ctrl.cpu().numpy()
    assert np.max(np.abs(got - ref_ctrl)) / np.max(np.abs(ref_ctrl)) <= 1e-4


def test_fit_step_batched_reduce_path_and_determinism():
    """B > 1 with several tiles per surface (workspace reduce + SGD in the update kernel)."""
    w = wl.surfaces("fitb", B=3, n=40, m=24, p=3, q=2, n_u=150, n_v=260, seed=31)
    rng = np.random.default_rng(3)
    Tf = (oracle.surface_fwd(w.ctrl, w.U, w.V, w.u, w.v, w.p, w.q)
          + rng.normal(0, 0.01, (3, 150, 260, 3))).astype(np.float32)
    lr = 50.0
    ref_loss, ref_grads, ref_ctrl = oracle_fit(w.ctrl, w, Tf.astype(np.float64), lr, 3)
    outs = []
    for _ in range(2):
        ctrl = T(w.ctrl)
        fitter = nb.SurfaceFitter(ctrl, T(w.U), T(w.V), T(w.u), T(w.v), T(Tf), w.p, w.q, lr)
        losses = fitter.run(3, graph=False).cpu().numpy()
        outs.append((losses, ctrl.cpu().numpy(), fitter.grad.cpu().numpy()))
    np.testing.assert_array_equal(outs[0][1], outs[1][1])     # bitwise repeatable
    assert np.max(np.abs(outs[0][0] - ref_loss)) / np.max(ref_loss) <= 1e-4
    assert bwd_err(outs[0][2], ref_grads[-1], w.ctrl) <= BWD_TOL
    assert np.max(np.abs(outs[0][1] - ref_ctrl)) / np.max(np.abs(ref_ctrl)) <= 1e-4


# --------------------------------------------------------------------------- parametric derivatives (NEXT-3)
DER_TOL = 1e-4   # normwise: max|dS_gpu - dS_ref| / max|dS_ref| per surface (as R16 for gradients)


def der_err(gpu, ref):
    B = ref.shape[0]
    e = np.abs(gpu.reshape(B, -1) - ref.reshape(B, -1)).max(axis=1)
    return float(np.max(e / np.abs(ref.reshape(B, -1)).max(axis=1)))


@pytest.mark.parametrize("case", ["cfg2", "cfg4", "batched", "deg15", "deg52", "ragged", "sparse", "cfg5net"])
def test_surface_derivs_parity(case):
    w = {"cfg2": lambda: wl.config2(),
         "cfg4": lambda: wl.config4(B=6),
         "batched": lambda: wl.config4(B=5, knots_batched=True),
         "deg15": lambda: wl.surfaces("d15", B=2, n=9, m=11, p=1, q=5, n_u=40, n_v=70, seed=3),
         "deg52": lambda: wl.surfaces("d52", B=2, n=11, m=7, p=5, q=2, n_u=33, n_v=130, seed=4),
         "ragged": lambda: wl.surfaces("dr", B=2, n=10, m=9, p=3, q=3, n_u=45, n_v=301, seed=5),
         "sparse": lambda: wl.surfaces("dsp", B=1, n=50, m=40, p=3, q=2, n_u=9, n_v=7, seed=6),
         "cfg5net": lambda: wl.config5(n_u=700, n_v=600)}[case]()
    S, Su, Sv, nrm = nb.surface_derivs(T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v), w.p, w.q)
    torch.cuda.synchronize()
    rS, rSu, rSv = oracle.surface_derivs(w.ctrl, w.U, w.V, w.u, w.v, w.p, w.q, w.knots_batched)
    assert fwd_err(S.cpu().numpy(), rS, w.ctrl) <= FWD_TOL
    assert der_err(Su.cpu().numpy(), rSu) <= DER_TOL
    assert der_err(Sv.cpu().numpy(), rSv) <= DER_TOL
    rn = np.cross(rSu, rSv)
    rn /= np.linalg.norm(rn, axis=-1, keepdims=True)
    cos = np.sum(nrm.cpu().numpy() * rn, axis=-1)
    assert np.min(cos) >= 1 - 1e-4


def test_surface_derivs_full_cfg4_sampled():
    """The derivative kernel in the bench launch configuration (config 4: 4096 surfaces, 128^2):
    32 sampled whole surfaces against the fp64 oracle (S, S_u, S_v, normals), every normal of
    the batch of unit length, and S equal to the grid forward's within the forward tolerance."""
    w = wl.config4()
    ctrl, U, V, u, v = T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v)
    S, Su, Sv, nrm = nb.surface_derivs(ctrl, U, V, u, v, w.p, w.q)
    Sf = nb.surface_fwd(ctrl, U, V, u, v, w.p, w.q)
    torch.cuda.synchronize()
    nlen = torch.linalg.vector_norm(nrm, dim=-1)
    assert float((nlen - 1).abs().max()) <= 1e-5
    idx = np.random.default_rng(9).choice(w.B, 32, replace=False)
    c = w.ctrl[idx]
    Sn = S.cpu().numpy()
    assert fwd_err(Sn, Sf.cpu().numpy(), w.ctrl) <= FWD_TOL
    parts = oracle.pmap(lambda k0, k1: oracle.surface_derivs(c[k0:k1], w.U, w.V, w.u, w.v, w.p, w.q),
                        [(k, k + 4) for k in range(0, 32, 4)])
    rS, rSu, rSv = (np.concatenate([pt[j] for pt in parts]) for j in range(3))
    assert fwd_err(Sn[idx], rS, c, "derivs cfg4 full") <= FWD_TOL
    e_u, e_v = der_err(Su.cpu().numpy()[idx], rSu), der_err(Sv.cpu().numpy()[idx], rSv)
    record("derivs cfg4 full", "Su", e_u); record("derivs cfg4 full", "Sv", e_v)
    assert e_u <= DER_TOL and e_v <= DER_TOL
    rn = np.cross(rSu, rSv)
    rn /= np.linalg.norm(rn, axis=-1, keepdims=True)
    assert np.min(np.sum(nrm.cpu().numpy()[idx] * rn, axis=-1)) >= 1 - 1e-4


def test_cylinder_normals_on_gpu():
    s2 = np.float32(np.sqrt(2.0) / 2.0)
    arc = [((1, 0), 1.0), ((1, 1), s2), ((0, 1), 1.0)]
    ctrl = np.zeros((1, 3, 2, 4), dtype=np.float32)
    for i, ((x, y), wgt) in enumerate(arc):
        for j, z in enumerate([0.0, 2.0]):
            ctrl[0, i, j] = [x, y, z, wgt]
    U = np.array([0, 0, 0, 1, 1, 1], np.float32)
    V = np.array([0, 0, 1, 1], np.float32)
    S, Su, Sv, nrm = nb.surface_derivs(T(ctrl), T(U), T(V), T(wl.uniform_grid(65)), T(wl.uniform_grid(9)), 2, 1)
    S, nrm = S.cpu().numpy().astype(np.float64), nrm.cpu().numpy().astype(np.float64)
    radial = S.copy(); radial[..., 2] = 0
    radial /= np.linalg.norm(radial, axis=-1, keepdims=True)
    assert np.max(np.abs(np.abs(np.sum(nrm * radial, axis=-1)) - 1.0)) <= 1e-5
