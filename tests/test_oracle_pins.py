"""Pins for the CPU oracle (oracle/): every oracle function is checked against something
other than itself — values the paper/SPEC print (tests/golden/, cited), closed forms
(Bernstein, uniform cubic, exact rational circle/cylinder), brute force (dense Eq.4/5
recursion, linear-scan FindSpan, dense Jacobian), invariants that follow from Eq.3/8/9,
and central finite differences. CPU only (no GPU marker)."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import workloads as wl

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SQ2 = math.sqrt(2.0) / 2.0


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def linear_scan_span(n, p, U, u):
    """Brute force of reading R3/R4: max{s in [p, n-1] : U[s] <= u and U[s] < U[s+1]}."""
    best = -1
    for s in range(p, n):
        if U[s] <= u and U[s] < U[s + 1]:
            best = s
    return best


def random_knots(rng, n, p, repeat=True):
    inner = np.sort(rng.uniform(0.05, 0.95, size=n - p - 1))
    if repeat and n - p - 1 >= 2:
        k = rng.integers(0, n - p - 2)
        mult = rng.integers(1, p + 1)           # interior multiplicity <= p
        for t in range(1, mult):
            if k + t < len(inner):
                inner[k + t] = inner[k]
        inner = np.sort(inner)
    return np.concatenate([np.zeros(p + 1), inner, np.ones(p + 1)])


def adversarial_params(U, rng, extra=20):
    vals = set([0.0, 1.0])
    for k in U:
        vals.add(float(k))
        vals.add(float(np.nextafter(k, 2.0)))
        vals.add(float(np.nextafter(k, -1.0)))
    vals |= set(rng.uniform(0, 1, size=extra).tolist())
    return sorted(v for v in vals if 0.0 <= v <= 1.0)


# ------------------------------------------------------------------------------ FindSpan
def test_find_span_golden():
    for c in load("find_span.json")["cases"]:
        assert oracle.find_span(c["n"], c["p"], c["U"], c["u"]) == c["span"], c


def test_find_span_equals_linear_scan():
    rng = np.random.default_rng(0)
    for trial in range(60):
        p = int(rng.integers(1, 6))
        n = int(rng.integers(p + 1, p + 12))
        U = random_knots(rng, n, p)
        for u in adversarial_params(U, rng):
            assert oracle.find_span(n, p, U, u) == linear_scan_span(n, p, U, u), (n, p, U, u)
    # fp32 config grids against fp32 clamped-uniform knots (exact-knot hits in cfg1: a=33, 66)
    for n, p, n_u in [(6, 3, 100), (8, 3, 64), (32, 3, 512), (16, 3, 128), (256, 3, 2049)]:
        U = wl.clamped_uniform_knots(n, p).astype(np.float64)
        u = wl.uniform_grid(n_u).astype(np.float64)
        sp, _ = oracle.spans(n, p, U, u)
        assert [linear_scan_span(n, p, U, x) for x in u] == sp.tolist()
    U = wl.clamped_uniform_knots(6, 3).astype(np.float64)
    u = wl.uniform_grid(100).astype(np.float64)
    assert u[33] == U[4] and u[66] == U[5]        # R2: config 1 hits interior knots exactly
    assert oracle.find_span(6, 3, U, u[33]) == 4 and oracle.find_span(6, 3, U, u[66]) == 5


def test_find_span_empty_last_interval():
    """R3: U[n-1] == U[n] (end multiplicity p+2) — the span at u = U[n] must step down to the
    last non-empty interval; its basis is the left limit (partition of unity, finite)."""
    n, p = 5, 2
    U = [0, 0, 0, 0.5, 1, 1, 1, 1]
    for u in (1.0, 0.75, 0.5, 0.0):
        assert oracle.find_span(n, p, U, u) == linear_scan_span(n, p, U, u)
    s = oracle.find_span(n, p, U, 1.0)
    assert s == 3
    N = oracle.basis_funs(s, 1.0, p, U)
    assert np.all(np.isfinite(N)) and abs(N.sum() - 1) < 1e-15
    np.testing.assert_allclose(oracle.basis_dense(n, p, U, 1.0)[s - p:s + 1], N, atol=1e-15)


def test_find_span_out_of_domain():
    U = [0, 0, 0, 0.5, 1, 1, 1]
    assert oracle.find_span(4, 2, U, -1e-9) == -1
    assert oracle.find_span(4, 2, U, 1.0 + 1e-9) == -1


# ------------------------------------------------------------------------------ basis
def test_basis_golden():
    for c in load("basis.json")["cases"]:
        s = oracle.find_span(c["n"], c["p"], c["U"], c["u"])
        assert s == c["span"]
        np.testing.assert_allclose(oracle.basis_funs(s, c["u"], c["p"], c["U"]), c["N"], rtol=0, atol=1e-15)


def test_basis_partition_of_unity_and_nonnegative():
    rng = np.random.default_rng(1)
    for trial in range(60):
        p = int(rng.integers(1, 6))
        n = int(rng.integers(p + 1, p + 12))
        U = random_knots(rng, n, p)
        for u in adversarial_params(U, rng):
            s = oracle.find_span(n, p, U, u)
            N = oracle.basis_funs(s, u, p, U)
            assert np.all(N >= 0.0)
            assert abs(N.sum() - 1.0) <= 1e-14


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_basis_bernstein_closed_form(p):
    U = [0.0] * (p + 1) + [1.0] * (p + 1)
    for u in np.linspace(0, 1, 37):
        s = oracle.find_span(p + 1, p, U, u)
        assert s == p
        N = oracle.basis_funs(s, u, p, U)
        ref = [math.comb(p, i) * u ** i * (1 - u) ** (p - i) for i in range(p + 1)]
        np.testing.assert_allclose(N, ref, rtol=0, atol=1e-15)


def test_basis_uniform_cubic_closed_form():
    n, p = 19, 3                                     # 16 spans, knots k/16 exact in binary
    U = np.concatenate([np.zeros(p), np.arange(17) / 16.0, np.ones(p)])
    assert len(U) == n + p + 1
    checked = 0
    for u in np.linspace(0, 1, 401):
        s = oracle.find_span(n, p, U, u)
        if not (2 * p <= s <= n - p - 1):            # all four N_{s-3..s} on uniform knots
            continue
        t = (u - U[s]) / (U[s + 1] - U[s])
        ref = np.array([(1 - t) ** 3, 3 * t ** 3 - 6 * t ** 2 + 4, -3 * t ** 3 + 3 * t ** 2 + 3 * t + 1, t ** 3]) / 6
        np.testing.assert_allclose(oracle.basis_funs(s, u, p, U), ref, rtol=0, atol=1e-13)
        checked += 1
    assert checked > 100


def test_dense_recursion_equals_local():
    rng = np.random.default_rng(2)
    for trial in range(50):
        p = int(rng.integers(1, 6))
        n = int(rng.integers(p + 1, p + 10))
        U = random_knots(rng, n, p)
        for u in adversarial_params(U, rng, 10):
            s = oracle.find_span(n, p, U, u)
            local = np.zeros(n)
            local[s - p:s + 1] = oracle.basis_funs(s, u, p, U)
            np.testing.assert_allclose(oracle.basis_dense(n, p, U, u), local, rtol=0, atol=1e-14)


def test_closed_eq5_reading_double_counts_interior_knots():
    """Why R2 (half-open Eq.5): under the printed closed interval u_i <= u <= u_{i+1}, two
    degree-0 functions are 1 at an interior knot, so the basis sums to 2 (SURVEY App.A ch.6)."""
    U = wl.clamped_uniform_knots(6, 3).astype(np.float64)
    u = float(U[4])
    closed = [1.0 if U[i] <= u <= U[i + 1] else 0.0 for i in range(len(U) - 1)]
    assert sum(closed) == 2.0
    assert abs(oracle.basis_dense(6, 3, U, u).sum() - 1.0) < 1e-15


# ------------------------------------------------------------------------------ points
def test_quarter_circle_golden_and_radius():
    g = load("circle.json")
    ctrl = np.array([g["ctrl"]])
    out = oracle.curve_fwd(ctrl, g["U"], [g["u"]], g["p"])
    np.testing.assert_allclose(out[0, 0], g["point"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(out[0, 0, :2], g["printed"], rtol=0, atol=5e-6)
    u = np.linspace(0, 1, 1000)
    out = oracle.curve_fwd(ctrl, g["U"], u, g["p"])
    r = np.hypot(out[0, :, 0], out[0, :, 1])
    assert np.max(np.abs(r - 1.0)) <= 1e-12


def full_circle():
    U = [0, 0, 0, .25, .25, .5, .5, .75, .75, 1, 1, 1]
    P = [(1, 0), (1, 1), (0, 1), (-1, 1), (-1, 0), (-1, -1), (0, -1), (1, -1), (1, 0)]
    w = [1, SQ2, 1, SQ2, 1, SQ2, 1, SQ2, 1]
    ctrl = np.array([[[x, y, 0.0, ww] for (x, y), ww in zip(P, w)]])
    return ctrl, U


def test_full_circle_repeated_knots():
    ctrl, U = full_circle()
    u = np.concatenate([np.linspace(0, 1, 997), [0.25, 0.5, 0.75]])
    out = oracle.curve_fwd(ctrl, U, u, 2)
    r = np.hypot(out[0, :, 0], out[0, :, 1])
    assert np.max(np.abs(r - 1.0)) <= 1e-12
    np.testing.assert_allclose(out[0, -3:, :2], [[0, 1], [-1, 0], [0, -1]], atol=1e-15)


def test_cylinder_patch():
    """Quarter arc (u, p=2) x line (v, q=1): x^2+y^2 = 1 and z = 2v exactly."""
    arc = [((1, 0), 1.0), ((1, 1), SQ2), ((0, 1), 1.0)]
    ctrl = np.zeros((1, 3, 2, 4))
    for i, ((x, y), w) in enumerate(arc):
        for j, z in enumerate([0.0, 2.0]):
            ctrl[0, i, j] = [x, y, z, w]
    u = np.linspace(0, 1, 33)
    v = np.linspace(0, 1, 17)
    out = oracle.surface_fwd(ctrl, [0, 0, 0, 1, 1, 1], [0, 0, 1, 1], u, v, 2, 1)
    r = np.hypot(out[0, ..., 0], out[0, ..., 1])
    assert np.max(np.abs(r - 1.0)) <= 1e-12
    np.testing.assert_allclose(out[0, :, :, 2], np.broadcast_to(2 * v, (33, 17)), atol=1e-14)


@pytest.mark.parametrize("c", [1.0, 0.37, 3.0])
def test_bernstein_surface_and_equal_weights(c):
    """No interior knots: S = sum B_i^p(u) B_j^q(v) P_ij (tensor Bezier) for any equal
    weights c (P:171 B-spline mode). p != q, n_u != n_v pins index order/layout."""
    rng = np.random.default_rng(3)
    p, q = 2, 3
    ctrl = np.zeros((1, p + 1, q + 1, 4))
    ctrl[0, ..., :3] = rng.normal(size=(p + 1, q + 1, 3))
    ctrl[0, ..., 3] = c
    u = np.linspace(0, 1, 7)
    v = np.linspace(0, 1, 5)
    out = oracle.surface_fwd(ctrl, [0] * (p + 1) + [1] * (p + 1), [0] * (q + 1) + [1] * (q + 1), u, v, p, q)
    Bu = np.array([[math.comb(p, i) * x ** i * (1 - x) ** (p - i) for i in range(p + 1)] for x in u])
    Bv = np.array([[math.comb(q, j) * y ** j * (1 - y) ** (q - j) for j in range(q + 1)] for y in v])
    ref = np.einsum("ai,bj,ijc->abc", Bu, Bv, ctrl[0, ..., :3])
    np.testing.assert_allclose(out[0], ref, rtol=0, atol=1e-14)


def random_surface(rng, B=1, p=None, q=None, n=None, m=None, n_u=None, n_v=None, batched=False):
    p = p or int(rng.integers(1, 4))
    q = q or int(rng.integers(1, 4))
    n = n or int(rng.integers(p + 1, p + 6))
    m = m or int(rng.integers(q + 1, q + 6))
    n_u = n_u or int(rng.integers(3, 9))
    n_v = n_v or int(rng.integers(3, 9))
    ctrl = np.empty((B, n, m, 4))
    ctrl[..., :3] = rng.uniform(-1, 1, size=(B, n, m, 3))
    ctrl[..., 3] = rng.uniform(0.5, 1.5, size=(B, n, m))
    if batched:
        U = np.stack([random_knots(rng, n, p) for _ in range(B)])
        V = np.stack([random_knots(rng, m, q) for _ in range(B)])
    else:
        U, V = random_knots(rng, n, p), random_knots(rng, m, q)
    u = np.sort(rng.uniform(0, 1, n_u)); u[0] = 0.0
    v = np.sort(rng.uniform(0, 1, n_v)); v[-1] = 1.0
    return ctrl, U, V, u, v, p, q


def test_constant_points_and_corner_interpolation():
    rng = np.random.default_rng(4)
    ctrl, U, V, u, v, p, q = random_surface(rng, n_u=6, n_v=7)
    c = np.array([0.3, -1.2, 2.5])
    const = ctrl.copy()
    const[..., :3] = c
    out = oracle.surface_fwd(const, U, V, u, v, p, q)
    np.testing.assert_allclose(out, np.broadcast_to(c, out.shape), rtol=0, atol=1e-15 * 4)
    out = oracle.surface_fwd(ctrl, U, V, [0.0, 1.0], [0.0, 1.0], p, q)
    P = ctrl[0, ..., :3]
    np.testing.assert_allclose(out[0, 0, 0], P[0, 0], atol=1e-15)
    np.testing.assert_allclose(out[0, 0, 1], P[0, -1], atol=1e-15)
    np.testing.assert_allclose(out[0, 1, 0], P[-1, 0], atol=1e-15)
    np.testing.assert_allclose(out[0, 1, 1], P[-1, -1], atol=1e-15)


def test_affine_invariance():
    rng = np.random.default_rng(5)
    ctrl, U, V, u, v, p, q = random_surface(rng, B=2, batched=True)
    A, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    t = rng.normal(size=3)
    moved = ctrl.copy()
    moved[..., :3] = ctrl[..., :3] @ A.T + t
    out = oracle.surface_fwd(ctrl, U, V, u, v, p, q, knots_batched=True)
    out2 = oracle.surface_fwd(moved, U, V, u, v, p, q, knots_batched=True)
    np.testing.assert_allclose(out2, out @ A.T + t, rtol=0, atol=1e-14)


def test_dense_forward_equals_local():
    rng = np.random.default_rng(6)
    for _ in range(20):
        ctrl, U, V, u, v, p, q = random_surface(rng)
        u = np.unique(np.concatenate([u, U[p:len(U) - p]]))      # include every knot
        dense, _ = oracle.surface_dense(ctrl[0], U, V, u, v, p, q)
        local = oracle.surface_fwd(ctrl, U, V, u, v, p, q)[0]
        np.testing.assert_allclose(local, dense, rtol=0, atol=1e-14)


# ------------------------------------------------------------------------------ backward
def loss_and_fd(ctrl, U, V, u, v, p, q, g, h=1e-6, batched=False):
    fd = np.zeros_like(ctrl)
    it = np.nditer(ctrl[..., 0], flags=["multi_index"])
    for _ in it:
        idx = it.multi_index
        for c in range(4):
            cp, cm = ctrl.copy(), ctrl.copy()
            cp[idx + (c,)] += h
            cm[idx + (c,)] -= h
            Lp = np.sum(oracle.surface_fwd(cp, U, V, u, v, p, q, batched) * g)
            Lm = np.sum(oracle.surface_fwd(cm, U, V, u, v, p, q, batched) * g)
            fd[idx + (c,)] = (Lp - Lm) / (2 * h)
    return fd


@pytest.mark.parametrize("seed", range(8))
def test_backward_finite_differences(seed):
    rng = np.random.default_rng(100 + seed)
    ctrl, U, V, u, v, p, q = random_surface(rng, B=2, batched=bool(seed % 2))
    batched = bool(seed % 2)
    g = rng.normal(size=(2, len(u), len(v), 3))
    fd = loss_and_fd(ctrl, U, V, u, v, p, q, g, batched=batched)
    for form in ("H", "E"):
        an = oracle.surface_bwd(ctrl, U, V, u, v, g, p, q, batched, form=form)
        assert np.max(np.abs(an - fd)) / np.max(np.abs(fd)) <= 1e-7, form


def test_form_e_equals_form_h_and_selected():
    rng = np.random.default_rng(7)
    for _ in range(10):
        ctrl, U, V, u, v, p, q = random_surface(rng, B=3, n_u=9, n_v=11)
        g = rng.normal(size=(3, len(u), len(v), 3))
        H = oracle.surface_bwd(ctrl, U, V, u, v, g, p, q, form="H")
        E = oracle.surface_bwd(ctrl, U, V, u, v, g, p, q, form="E")
        scale = np.max(np.abs(E))
        assert np.max(np.abs(H - E)) <= 1e-14 * scale * 10
        sel = [(k, i, j) for k in range(3) for i in range(ctrl.shape[1]) for j in range(ctrl.shape[2])]
        S = oracle.surface_bwd_selected(ctrl, U, V, u, v, g, p, q, sel)
        np.testing.assert_allclose(S.reshape(E.shape), E, rtol=0, atol=1e-13 * scale)


def test_dense_jacobian_transpose_and_sparsity():
    rng = np.random.default_rng(8)
    for _ in range(8):
        ctrl, U, V, u, v, p, q = random_surface(rng)
        # parameters strictly inside spans: every local basis value is non-zero
        inner_u = U[p:len(U) - p]
        u = np.array([x for x in u if np.min(np.abs(inner_u - x)) > 1e-3])
        inner_v = V[q:len(V) - q]
        v = np.array([y for y in v if np.min(np.abs(inner_v - y)) > 1e-3])
        if len(u) == 0 or len(v) == 0:
            continue
        out, J = oracle.surface_dense(ctrl[0], U, V, u, v, p, q, jacobian=True)
        g = rng.normal(size=(len(u), len(v), 3))
        dense_grad = (J.T @ g.reshape(-1)).reshape(ctrl.shape[1:])
        local = oracle.surface_bwd(ctrl, U, V, u, v, g[None], p, q, form="E")[0]
        np.testing.assert_allclose(local, dense_grad, rtol=0, atol=1e-13 * np.max(np.abs(dense_grad)))
        nnz = np.count_nonzero(J, axis=1)
        assert np.all(nnz == 2 * (p + 1) * (q + 1))


def test_backward_invariants():
    rng = np.random.default_rng(9)
    ctrl, U, V, u, v, p, q = random_surface(rng, B=1, n_u=13, n_v=10)
    g = rng.normal(size=(1, len(u), len(v), 3))
    G = oracle.surface_bwd(ctrl, U, V, u, v, g, p, q)[0]
    S = oracle.surface_fwd(ctrl, U, V, u, v, p, q)
    sc = np.sum(np.abs(g))
    # translation invariance: sum_ij dP_ij = sum_pts g      (Eq.8 summed)
    np.testing.assert_allclose(G[..., :3].sum(axis=(0, 1)), g[0].sum(axis=(0, 1)), atol=1e-13 * sc)
    # S homogeneous of degree 0 in w: sum_ij w_ij dw_ij = 0
    assert abs(np.sum(ctrl[0, ..., 3] * G[..., 3])) <= 1e-13 * sc
    # S linear in P: sum_ij P_ij . dP_ij = sum_pts g . S
    assert abs(np.sum(ctrl[0, ..., :3] * G[..., :3]) - np.sum(g * S)) <= 1e-13 * sc
    # g == 0 -> zero gradient exactly
    assert np.all(oracle.surface_bwd(ctrl, U, V, u, v, 0 * g, p, q) == 0.0)
    # constant control points -> dw == 0
    const = ctrl.copy(); const[..., :3] = [0.5, -0.25, 1.5]
    Gc = oracle.surface_bwd(const, U, V, u, v, g, p, q)
    assert np.max(np.abs(Gc[..., 3])) <= 1e-14 * sc


def test_unit_weights_unit_upstream():
    """w == 1, g == 1: dP_ij = (sum_a N_i(u_a)) (sum_b N_j(v_b)) per coordinate."""
    rng = np.random.default_rng(10)
    ctrl, U, V, u, v, p, q = random_surface(rng, n_u=11, n_v=9)
    ctrl[..., 3] = 1.0
    g = np.ones((1, len(u), len(v), 3))
    G = oracle.surface_bwd(ctrl, U, V, u, v, g, p, q)[0]
    n, m = ctrl.shape[1:3]
    su = sum(oracle.basis_dense(n, p, U, x) for x in u)
    sv = sum(oracle.basis_dense(m, q, V, y) for y in v)
    for c in range(3):
        np.testing.assert_allclose(G[..., c], np.outer(su, sv), rtol=0, atol=1e-13)


def test_curve_finite_differences_and_surface_equivalence():
    rng = np.random.default_rng(11)
    for p in (1, 2, 3, 5):
        n = p + 4
        U = random_knots(rng, n, p)
        ctrl = np.empty((2, n, 4)); ctrl[..., :3] = rng.uniform(-1, 1, (2, n, 3)); ctrl[..., 3] = rng.uniform(.5, 1.5, (2, n))
        u = np.sort(rng.uniform(0, 1, 17)); u[0], u[-1] = 0.0, 1.0
        g = rng.normal(size=(2, 17, 3))
        an = oracle.curve_bwd(ctrl, U, u, g, p)
        fd = np.zeros_like(ctrl); h = 1e-6
        for idx in np.ndindex(ctrl.shape):
            cp, cm = ctrl.copy(), ctrl.copy(); cp[idx] += h; cm[idx] -= h
            fd[idx] = (np.sum(oracle.curve_fwd(cp, U, u, p) * g) - np.sum(oracle.curve_fwd(cm, U, u, p) * g)) / (2 * h)
        assert np.max(np.abs(an - fd)) / np.max(np.abs(fd)) <= 1e-7
        # a curve is the surface with a trivial linear v-direction whose two rows coincide
        sctrl = np.repeat(ctrl[:, :, None, :], 2, axis=2)
        s = oracle.surface_fwd(sctrl, U, [0, 0, 1, 1], u, [0.0, 0.3, 1.0], p, 1)
        for b in range(3):
            np.testing.assert_allclose(s[:, :, b], oracle.curve_fwd(ctrl, U, u, p), atol=1e-14)


def test_error_paths():
    rng = np.random.default_rng(12)
    ctrl, U, V, u, v, p, q = random_surface(rng)
    bad = U.copy(); bad[p + 1], bad[p + 2] = 0.9, 0.1
    if len(U) > p + 3:
        with pytest.raises(oracle.OracleError):
            oracle.surface_fwd(ctrl, bad, V, u, v, p, q)
    with pytest.raises(oracle.OracleError):
        oracle.surface_fwd(ctrl, U, V, np.array([-0.1]), v, p, q)
    neg = ctrl.copy(); neg[0, 0, 0, 3] = 0.0
    with pytest.raises(oracle.OracleError):
        oracle.surface_fwd(neg, U, V, u, v, p, q)


# ------------------------------------------------------------------------------ NEXT-3: derivatives
def test_basis_ders_golden_and_sum_zero():
    for c in load("basis_ders.json")["cases"]:
        s = oracle.find_span(c["n"], c["p"], c["U"], c["u"])
        assert s == c["span"]
        np.testing.assert_allclose(oracle.basis_ders1(s, c["u"], c["p"], c["U"]), c["dN"], rtol=0, atol=1e-14)
    rng = np.random.default_rng(40)
    for _ in range(40):
        p = int(rng.integers(1, 6))
        n = int(rng.integers(p + 1, p + 10))
        U = random_knots(rng, n, p)
        for u in adversarial_params(U, rng, 10):
            s = oracle.find_span(n, p, U, u)
            assert abs(oracle.basis_ders1(s, u, p, U).sum()) <= 1e-10   # d/du (partition of unity)


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_basis_ders_bernstein_and_fd(p):
    U = [0.0] * (p + 1) + [1.0] * (p + 1)
    for u in np.linspace(0.01, 0.99, 23):
        d = oracle.basis_ders1(p, u, p, U)
        ref = [math.comb(p, i) * ((i * u ** (i - 1) if i else 0.0) * (1 - u) ** (p - i)
                                   - (u ** i) * ((p - i) * (1 - u) ** (p - i - 1) if p - i else 0.0))
               for i in range(p + 1)]
        np.testing.assert_allclose(d, ref, rtol=0, atol=1e-12)
    rng = np.random.default_rng(41 + p)
    n = p + 6
    U = random_knots(rng, n, p, repeat=False)
    h = 1e-7
    for u in rng.uniform(0.06, 0.94, 30):
        s = oracle.find_span(n, p, U, u)
        if oracle.find_span(n, p, U, u - h) != s or oracle.find_span(n, p, U, u + h) != s:
            continue
        fd = (oracle.basis_funs(s, u + h, p, U) - oracle.basis_funs(s, u - h, p, U)) / (2 * h)
        np.testing.assert_allclose(oracle.basis_ders1(s, u, p, U), fd, rtol=0, atol=1e-6)


def test_surface_derivs_fd_and_value():
    rng = np.random.default_rng(42)
    for _ in range(6):
        ctrl, U, V, u, v, p, q = random_surface(rng, B=2, batched=True)
        # keep samples away from knots so the central differences stay in one span
        u = np.array([x for x in np.linspace(0.03, 0.97, 9) if np.min(np.abs(U - x)) > 1e-4])
        v = np.array([y for y in np.linspace(0.04, 0.96, 7) if np.min(np.abs(V - y)) > 1e-4])
        S, Su, Sv = oracle.surface_derivs(ctrl, U, V, u, v, p, q, knots_batched=True)
        np.testing.assert_allclose(S, oracle.surface_fwd(ctrl, U, V, u, v, p, q, True), rtol=0, atol=1e-15)
        h = 1e-6
        fu = (oracle.surface_fwd(ctrl, U, V, u + h, v, p, q, True) - oracle.surface_fwd(ctrl, U, V, u - h, v, p, q, True)) / (2 * h)
        fv = (oracle.surface_fwd(ctrl, U, V, u, v + h, p, q, True) - oracle.surface_fwd(ctrl, U, V, u, v - h, p, q, True)) / (2 * h)
        assert np.max(np.abs(Su - fu)) <= 1e-6 * max(1.0, np.max(np.abs(Su)))
        assert np.max(np.abs(Sv - fv)) <= 1e-6 * max(1.0, np.max(np.abs(Sv)))


def test_cylinder_normals_radial_and_plane_normal():
    arc = [((1, 0), 1.0), ((1, 1), SQ2), ((0, 1), 1.0)]
    ctrl = np.zeros((1, 3, 2, 4))
    for i, ((x, y), w) in enumerate(arc):
        for j, z in enumerate([0.0, 2.0]):
            ctrl[0, i, j] = [x, y, z, w]
    u = np.linspace(0, 1, 21)
    v = np.linspace(0, 1, 5)
    S, Su, Sv = oracle.surface_derivs(ctrl, [0, 0, 0, 1, 1, 1], [0, 0, 1, 1], u, v, 2, 1)
    nrm = np.cross(Su, Sv)
    nrm /= np.linalg.norm(nrm, axis=-1, keepdims=True)
    radial = S.copy(); radial[..., 2] = 0
    np.testing.assert_allclose(np.abs(np.sum(nrm * radial, axis=-1)), 1.0, atol=1e-12)
    np.testing.assert_allclose(Sv[..., 2], 2.0, atol=1e-14)                             # z = 2v
    # planar bilinear patch at z = 0: normal (0, 0, 1); reversed v order flips it
    plane = np.zeros((1, 2, 2, 4)); plane[..., 3] = 1.0
    plane[0, :, :, 0] = [[0, 0], [1, 1]]; plane[0, :, :, 1] = [[0, 1], [0, 1]]
    _, pu, pv = oracle.surface_derivs(plane, [0, 0, 1, 1], [0, 0, 1, 1], [0.3], [0.6], 1, 1)
    np.testing.assert_allclose(np.cross(pu, pv)[0, 0, 0], [0, 0, 1], atol=1e-15)
    _, pu, pv = oracle.surface_derivs(plane[:, :, ::-1].copy(), [0, 0, 1, 1], [0, 0, 1, 1], [0.3], [0.6], 1, 1)
    np.testing.assert_allclose(np.cross(pu, pv)[0, 0, 0], [0, 0, -1], atol=1e-15)


# ---------------------------------------------------------------- NEXT-1: paired points
def random_uv(rng, U, V, p, q, B, N):
    """Scattered (u, v) in the domain, with knot hits and both ends mixed in."""
    uv = rng.uniform(0, 1, size=(B, N, 2))
    Ub = np.asarray(U).reshape(-1, np.shape(U)[-1])
    Vb = np.asarray(V).reshape(-1, np.shape(V)[-1])
    for k in range(B):
        Uk, Vk = Ub[k % len(Ub)], Vb[k % len(Vb)]
        hits = [(Uk[rng.integers(p, len(Uk) - p)], Vk[rng.integers(q, len(Vk) - q)]) for _ in range(N // 4)]
        for t, (a, b) in enumerate(hits):
            uv[k, 4 * t] = (a, b)
        if N >= 3:
            uv[k, 1] = (0.0, 1.0)
            uv[k, 2] = (1.0, 0.0)
    return uv


def test_points_at_grid_coordinates_equal_grid_oracle():
    """The grid is the special case uv[k][a*n_v+b] = (u_a, v_b): identical forward, and the
    same gradient (P:154-163 per point; the grid functions are pinned above)."""
    rng = np.random.default_rng(21)
    for trial in range(6):
        ctrl, U, V, u, v, p, q = random_surface(rng, B=2, batched=bool(trial % 2))
        uu, vv = np.meshgrid(u, v, indexing="ij")
        uv = np.broadcast_to(np.stack([uu.ravel(), vv.ravel()], -1), (2, uu.size, 2)).copy()
        out = oracle.surface_fwd_points(ctrl, U, V, uv, p, q, bool(trial % 2))
        ref = oracle.surface_fwd(ctrl, U, V, u, v, p, q, bool(trial % 2))
        assert np.array_equal(out, ref.reshape(2, -1, 3))
        g = rng.normal(size=(2, len(u), len(v), 3))
        G = oracle.surface_bwd_points(ctrl, U, V, uv, g.reshape(2, -1, 3), p, q, bool(trial % 2))
        E = oracle.surface_bwd(ctrl, U, V, u, v, g, p, q, bool(trial % 2), form="E")
        np.testing.assert_allclose(G, E, rtol=0, atol=1e-14 * np.max(np.abs(E)))


@pytest.mark.parametrize("seed", range(4))
def test_points_backward_finite_differences(seed):
    rng = np.random.default_rng(200 + seed)
    ctrl, U, V, _, _, p, q = random_surface(rng, B=2, batched=bool(seed % 2))
    uv = random_uv(rng, U, V, p, q, 2, 23)
    g = rng.normal(size=(2, 23, 3))
    an = oracle.surface_bwd_points(ctrl, U, V, uv, g, p, q, bool(seed % 2))
    fd = np.zeros_like(ctrl)
    h = 1e-6
    for idx in np.ndindex(ctrl.shape):
        cp, cm = ctrl.copy(), ctrl.copy()
        cp[idx] += h
        cm[idx] -= h
        fd[idx] = (np.sum(oracle.surface_fwd_points(cp, U, V, uv, p, q, bool(seed % 2)) * g)
                   - np.sum(oracle.surface_fwd_points(cm, U, V, uv, p, q, bool(seed % 2)) * g)) / (2 * h)
    assert np.max(np.abs(an - fd)) / np.max(np.abs(fd)) <= 1e-7


def test_points_dense_brute_force_and_cylinder():
    """Each paired point against the literal Eq.4/5 dense evaluation and its Jacobian J^T g
    (P:238), and the exact cylinder x^2 + y^2 = 1, z = 2v at scattered points."""
    rng = np.random.default_rng(22)
    for _ in range(4):
        ctrl, U, V, _, _, p, q = random_surface(rng, B=1)
        uv = random_uv(rng, U, V, p, q, 1, 9)
        g = rng.normal(size=(1, 9, 3))
        out = oracle.surface_fwd_points(ctrl, U, V, uv, p, q)
        G = oracle.surface_bwd_points(ctrl, U, V, uv, g, p, q)
        acc = np.zeros_like(G[0])
        for t in range(9):
            o, J = oracle.surface_dense(ctrl[0], U, V, uv[0, t, :1], uv[0, t, 1:], p, q, jacobian=True)
            np.testing.assert_allclose(out[0, t], o[0, 0], rtol=0, atol=1e-14)
            acc += (J.T @ g[0, t]).reshape(acc.shape)
        np.testing.assert_allclose(G[0], acc, rtol=0, atol=1e-13 * np.max(np.abs(acc)))
    arc = [((1, 0), 1.0), ((1, 1), SQ2), ((0, 1), 1.0)]
    cyl = np.zeros((1, 3, 2, 4))
    for i, ((x, y), w) in enumerate(arc):
        for j, z in enumerate([0.0, 2.0]):
            cyl[0, i, j] = [x, y, z, w]
    uv = rng.uniform(0, 1, size=(1, 200, 2))
    out = oracle.surface_fwd_points(cyl, [0, 0, 0, 1, 1, 1], [0, 0, 1, 1], uv, 2, 1)
    assert np.max(np.abs(np.hypot(out[0, :, 0], out[0, :, 1]) - 1.0)) <= 1e-12
    np.testing.assert_allclose(out[0, :, 2], 2 * uv[0, :, 1], atol=1e-14)


def test_points_backward_invariants_and_errors():
    rng = np.random.default_rng(23)
    ctrl, U, V, _, _, p, q = random_surface(rng, B=1)
    uv = random_uv(rng, U, V, p, q, 1, 40)
    g = rng.normal(size=(1, 40, 3))
    G = oracle.surface_bwd_points(ctrl, U, V, uv, g, p, q)[0]
    S = oracle.surface_fwd_points(ctrl, U, V, uv, p, q)
    sc = np.sum(np.abs(g))
    np.testing.assert_allclose(G[..., :3].sum(axis=(0, 1)), g[0].sum(axis=0), atol=1e-13 * sc)
    assert abs(np.sum(ctrl[0, ..., 3] * G[..., 3])) <= 1e-13 * sc
    assert abs(np.sum(ctrl[0, ..., :3] * G[..., :3]) - np.sum(g * S)) <= 1e-13 * sc
    bad = uv.copy(); bad[0, 5, 1] = 1.5
    with pytest.raises(oracle.OracleError):
        oracle.surface_fwd_points(ctrl, U, V, bad, p, q)
    assert oracle.surface_fwd_points(ctrl, U, V, uv[:, :0], p, q).shape == (1, 0, 3)


# ---------------------------------------------------------------- NEXT-4: knot gradients
def distinct_knots(rng, n, p, lo=0.0, hi=1.0):
    inner = np.sort(rng.uniform(0.1, 0.9, n - p - 1))
    while n - p - 1 > 1 and np.min(np.diff(inner)) < 0.03:
        inner = np.sort(rng.uniform(0.1, 0.9, n - p - 1))
    return np.concatenate([[lo] * (p + 1), inner, [hi] * (p + 1)])


def params_away_from(U, rng, k, margin=0.01):
    out = []
    while len(out) < k:
        x = rng.uniform(0.02, 0.98)
        if np.min(np.abs(np.asarray(U) - x)) > margin:
            out.append(x)
    return np.sort(np.array(out))


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_basis_knot_derivative_fd(p):
    rng = np.random.default_rng(300 + p)
    n = p + 5
    U = distinct_knots(rng, n, p)
    h = 1e-7
    for u in params_away_from(U, rng, 6):
        for kk in range(n + p + 1):
            fd, tol = fd_knot(lambda K_: oracle.basis_dense(n, p, K_, u), U, (kk,), h)
            if fd is None:
                continue
            an = oracle.basis_dknot(n, p, U, u, kk)
            assert np.max(np.abs(an - fd)) <= tol * max(1.0, np.max(np.abs(fd))), (kk, u)


def fd_knot(f, K, idx, h):
    """Central difference in knot K[idx] when both K +- h keep the vector non-decreasing,
    else the one-sided difference that does (looser tolerance), else None."""
    row = K[idx[:-1]] if K.ndim == 2 else K
    k = idx[-1]
    up_ok = k + 1 >= len(row) or row[k] + h <= row[k + 1]
    dn_ok = k == 0 or row[k] - h >= row[k - 1]
    Kp, Km = K.copy(), K.copy()
    Kp[idx] += h
    Km[idx] -= h
    if up_ok and dn_ok:
        return (f(Kp) - f(Km)) / (2 * h), 1e-6
    if up_ok:
        return (f(Kp) - f(K)) / h, 2e-5
    if dn_ok:
        return (f(K) - f(Km)) / h, 2e-5
    return None, None


@pytest.mark.parametrize("seed", range(4))
def test_surface_knot_grad_fd_and_invariants(seed):
    rng = np.random.default_rng(400 + seed)
    B, p, q = 2, 1 + seed % 3, 1 + (seed + 1) % 3
    n, m = p + 3 + seed % 2, q + 4
    batched = bool(seed % 2)
    if batched:
        U = np.stack([distinct_knots(rng, n, p) for _ in range(B)])
        V = np.stack([distinct_knots(rng, m, q) for _ in range(B)])
        allU, allV = U.ravel(), V.ravel()
    else:
        U, V = distinct_knots(rng, n, p), distinct_knots(rng, m, q)
        allU, allV = U, V
    u = params_away_from(allU, rng, 7)
    v = params_away_from(allV, rng, 5)
    ctrl = np.empty((B, n, m, 4))
    ctrl[..., :3] = rng.uniform(-1, 1, (B, n, m, 3))
    ctrl[..., 3] = rng.uniform(0.5, 1.5, (B, n, m))
    g = rng.normal(size=(B, len(u), len(v), 3))
    gU, gV = oracle.surface_knot_grad(ctrl, U, V, u, v, g, p, q, batched)
    h = 1e-7
    L = lambda U_, V_: np.sum(oracle.surface_fwd(ctrl, U_, V_, u, v, p, q, batched) * g)
    for which, K, G in (("U", U, gU), ("V", V, gV)):
        for idx in np.ndindex(K.shape):
            fd, tol = fd_knot(lambda K_: L(K_, V) if which == "U" else L(U, K_), K, idx, h)
            if fd is None:
                continue  # an inner copy of a clamped end knot: no order-preserving perturbation
            gi = G[idx] if batched else G[0][idx]
            assert abs(gi - fd) <= tol * max(1.0, np.max(np.abs(G))), (which, idx)
    # translating all knots of a direction by d moves the parameters by -d (shift invariance):
    # sum_k dL/dU_k = -sum g . S_u;  scaling knots and parameters together: sum_k U_k dL/dU_k = -sum u g . S_u
    _, Su, Sv = oracle.surface_derivs(ctrl, U, V, u, v, p, q, batched)
    gs = np.sum(g * Su, axis=(2, 3))            # [B][n_u]
    gsv = np.sum(g * Sv, axis=(1, 3))           # [B][n_v]
    sc = np.sum(np.abs(g)) * 10
    if batched:
        np.testing.assert_allclose(gU.sum(axis=1), -gs.sum(axis=1), atol=1e-12 * sc)
        np.testing.assert_allclose((gU * U).sum(axis=1), -(gs * u).sum(axis=1), atol=1e-12 * sc)
        np.testing.assert_allclose(gV.sum(axis=1), -gsv.sum(axis=1), atol=1e-12 * sc)
    else:
        assert abs(gU.sum() + gs.sum()) <= 1e-12 * sc
        assert abs((gU[0] * U).sum() + (gs * u).sum()) <= 1e-12 * sc
        assert abs(gV.sum() + gsv.sum()) <= 1e-12 * sc
        assert abs((gV[0] * V).sum() + (gsv * v).sum()) <= 1e-12 * sc


def test_curve_knot_grad_fd():
    rng = np.random.default_rng(500)
    for p in (1, 2, 3, 4):
        n = p + 4
        U = distinct_knots(rng, n, p)
        u = params_away_from(U, rng, 9)
        ctrl = np.empty((2, n, 4))
        ctrl[..., :3] = rng.uniform(-1, 1, (2, n, 3))
        ctrl[..., 3] = rng.uniform(0.5, 1.5, (2, n))
        g = rng.normal(size=(2, len(u), 3))
        gU = oracle.curve_knot_grad(ctrl, U, u, g, p)[0]
        h = 1e-7
        for kk in range(n + p + 1):
            fd, tol = fd_knot(lambda K_: np.sum(oracle.curve_fwd(ctrl, K_, u, p) * g), U, (kk,), h)
            if fd is not None:
                assert abs(gU[kk] - fd) <= tol * max(1.0, np.max(np.abs(gU)))
