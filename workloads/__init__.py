"""Seeded synthetic inputs for the NURBS-Diff hot path (DESIGN.md §4 "input recipe").

This module holds no arithmetic of the method: it only builds knot vectors, parameter grids,
control nets, weights and upstream gradients as fp32 numpy arrays. The SAME arrays feed the
CUDA path and the oracle. Generator: numpy PCG64, seed = config number unless given.

Shapes follow BASELINE.json `configs` and SURVEY.md §8(d):
  cfg1  cubic curve, 6 ctrl, clamped uniform knots, 100 samples
  cfg2  bicubic 8x8 net, random weights, 64x64 grid
  cfg3  bicubic 32x32 net, 512x512 grid (fitting workload)
  cfg4  4096 bicubic 16x16 nets, 128x128 grid (decoder batch)
  cfg5  one bicubic 256x256 net, 8192x8192 grid
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

f32 = np.float32


def clamped_uniform_knots(n: int, p: int) -> np.ndarray:
    """Clamped uniform knot vector (reading R7): p+1 zeros, fp32(k)/fp32(n-p) for k=1..n-p-1,
    p+1 ones. Length n+p+1."""
    inner = [f32(k) / f32(n - p) for k in range(1, n - p)]
    return np.array([0.0] * (p + 1) + inner + [1.0] * (p + 1), dtype=f32)


def random_clamped_knots(rng: np.random.Generator, n: int, p: int, min_gap: float = 0.0) -> np.ndarray:
    """Clamped knots with sorted random interior knots (per-surface knots, Alg.1 U_k)."""
    inner = np.sort(rng.uniform(0.02, 0.98, size=n - p - 1).astype(f32))
    return np.concatenate([np.zeros(p + 1, f32), inner, np.ones(p + 1, f32)]).astype(f32)


def uniform_grid(n_s: int) -> np.ndarray:
    """Inclusive uniform samples of [0,1] (reading R8): fp32(a)/fp32(n_s-1); n_s==1 -> [0]."""
    if n_s == 1:
        return np.zeros(1, dtype=f32)
    return (np.arange(n_s, dtype=f32) / f32(n_s - 1)).astype(f32)


def lattice_net(rng: np.random.Generator, B: int, n: int, m: int, sigma: float = 0.1,
                wlo: float = 0.5, whi: float = 1.5) -> np.ndarray:
    """ctrl[B][n][m][4] = (i/(n-1), j/(m-1), 0) + N(0, sigma)^3, w ~ U(wlo, whi) (R15)."""
    ii, jj = np.meshgrid(np.arange(n, dtype=f32) / f32(max(n - 1, 1)),
                         np.arange(m, dtype=f32) / f32(max(m - 1, 1)), indexing="ij")
    ctrl = np.empty((B, n, m, 4), dtype=f32)
    ctrl[..., 0] = ii
    ctrl[..., 1] = jj
    ctrl[..., 2] = 0.0
    ctrl[..., :3] += rng.normal(0.0, sigma, size=(B, n, m, 3)).astype(f32)
    ctrl[..., 3] = rng.uniform(wlo, whi, size=(B, n, m)).astype(f32)
    return ctrl


def random_net(rng: np.random.Generator, shape, wlo: float = 0.5, whi: float = 1.5) -> np.ndarray:
    ctrl = np.empty(tuple(shape) + (4,), dtype=f32)
    ctrl[..., :3] = rng.uniform(-1.0, 1.0, size=tuple(shape) + (3,)).astype(f32)
    ctrl[..., 3] = rng.uniform(wlo, whi, size=tuple(shape)).astype(f32)
    return ctrl


def normal(rng: np.random.Generator, shape) -> np.ndarray:
    return rng.standard_normal(size=shape, dtype=f32)


@dataclass
class Surfaces:
    """One synthetic surface workload (all fp32, C-contiguous)."""
    name: str
    p: int
    q: int
    ctrl: np.ndarray          # [B][n][m][4]
    U: np.ndarray             # [n+p+1] or [B][n+p+1]
    V: np.ndarray
    u: np.ndarray             # [n_u]
    v: np.ndarray             # [n_v]
    knots_batched: bool = False
    extra: dict = field(default_factory=dict)

    @property
    def B(self): return self.ctrl.shape[0]
    @property
    def n(self): return self.ctrl.shape[1]
    @property
    def m(self): return self.ctrl.shape[2]
    @property
    def n_u(self): return len(self.u)
    @property
    def n_v(self): return len(self.v)
    @property
    def points(self): return self.B * self.n_u * self.n_v

    def grad_out(self, seed: int | None = None) -> np.ndarray:
        rng = np.random.default_rng(seed if seed is not None else 1000 + sum(self.name.encode()))
        return normal(rng, (self.B, self.n_u, self.n_v, 3))


@dataclass
class Curves:
    name: str
    p: int
    ctrl: np.ndarray          # [B][n][4]
    U: np.ndarray
    u: np.ndarray
    knots_batched: bool = False

    @property
    def B(self): return self.ctrl.shape[0]
    @property
    def n(self): return self.ctrl.shape[1]
    @property
    def n_u(self): return len(self.u)

    def grad_out(self, seed: int = 11) -> np.ndarray:
        return normal(np.random.default_rng(seed), (self.B, self.n_u, 3))


def config1(seed: int = 1) -> Curves:
    rng = np.random.default_rng(seed)
    n, p = 6, 3
    return Curves("cfg1", p, random_net(rng, (1, n)), clamped_uniform_knots(n, p), uniform_grid(100))


def surfaces(name: str, B: int, n: int, m: int, p: int, q: int, n_u: int, n_v: int, seed: int,
             knots_batched: bool = False, sigma: float = 0.1) -> Surfaces:
    rng = np.random.default_rng(seed)
    ctrl = lattice_net(rng, B, n, m, sigma)
    if knots_batched:
        U = np.stack([random_clamped_knots(rng, n, p) for _ in range(B)])
        V = np.stack([random_clamped_knots(rng, m, q) for _ in range(B)])
    else:
        U, V = clamped_uniform_knots(n, p), clamped_uniform_knots(m, q)
    return Surfaces(name, p, q, ctrl, U, V, uniform_grid(n_u), uniform_grid(n_v), knots_batched)


def config2(seed: int = 2) -> Surfaces:
    return surfaces("cfg2", 1, 8, 8, 3, 3, 64, 64, seed)


def config3(seed: int = 3) -> Surfaces:
    return surfaces("cfg3", 1, 32, 32, 3, 3, 512, 512, seed)


def config3_fit(seed: int = 3, n: int = 32, n_s: int = 512):
    """Config 3 (SGD surface fit, §4.2): a ground-truth NURBS (lattice + N(0,0.1),
    w* ~ U(0.5,1.5)) whose surface is the target, and the initial guess P* + N(0, 0.05), w = 1
    (SURVEY §8(d)). Returns (truth, init) Surfaces; the target points are computed by the caller."""
    truth = surfaces("cfg3_truth", 1, n, n, 3, 3, n_s, n_s, seed)
    rng = np.random.default_rng(seed + 100)
    init_ctrl = truth.ctrl.copy()
    init_ctrl[..., :3] += rng.normal(0.0, 0.05, size=init_ctrl[..., :3].shape).astype(f32)
    init_ctrl[..., 3] = 1.0
    init = Surfaces("cfg3_init", 3, 3, init_ctrl, truth.U, truth.V, truth.u, truth.v)
    return truth, init


def config4(seed: int = 4, B: int = 4096, knots_batched: bool = False) -> Surfaces:
    return surfaces("cfg4", B, 16, 16, 3, 3, 128, 128, seed, knots_batched)


def config5(seed: int = 5, n_u: int = 8192, n_v: int = 8192) -> Surfaces:
    return surfaces("cfg5", 1, 256, 256, 3, 3, n_u, n_v, seed)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


@dataclass
class PairedSurfaces:
    """Paired (scattered) parameter points (NEXT-1): point t of surface k sits at uv[k][t]."""
    name: str
    p: int
    q: int
    ctrl: np.ndarray          # [B][n][m][4]
    U: np.ndarray             # [n+p+1] or [B][n+p+1]
    V: np.ndarray
    uv: np.ndarray            # [B][N][2]
    knots_batched: bool = False

    @property
    def B(self): return self.ctrl.shape[0]
    @property
    def n(self): return self.ctrl.shape[1]
    @property
    def m(self): return self.ctrl.shape[2]
    @property
    def N(self): return self.uv.shape[1]
    @property
    def points(self): return self.B * self.N

    def grad_out(self, seed: int | None = None) -> np.ndarray:
        rng = np.random.default_rng(seed if seed is not None else 2000 + sum(self.name.encode()))
        return normal(rng, (self.B, self.N, 3))


def paired(name: str, B: int, n: int, m: int, p: int, q: int, N: int, seed: int,
           knots_batched: bool = False, knot_hits: bool = True) -> PairedSurfaces:
    """Lattice nets (as `surfaces`) with N scattered points per surface, uv ~ U(0,1)^2 in fp32
    (point-cloud parameters, SplineNet/ParSeNet style). With `knot_hits`, every 16th
    point is moved onto a knot pair and points 1, 2 onto the corners (0,1), (1,0)."""
    base = surfaces(name, B, n, m, p, q, 1, 1, seed, knots_batched)
    rng = np.random.default_rng(seed + 7)
    uv = rng.uniform(0.0, 1.0, size=(B, N, 2)).astype(f32)
    if knot_hits and N > 0:
        Ub = base.U.reshape(-1, base.U.shape[-1])
        Vb = base.V.reshape(-1, base.V.shape[-1])
        t = np.arange(0, N, 16)
        for k in range(B):
            Uk, Vk = Ub[k % len(Ub)], Vb[k % len(Vb)]
            uv[k, t, 0] = Uk[rng.integers(p, len(Uk) - p, size=len(t))]
            uv[k, t, 1] = Vk[rng.integers(q, len(Vk) - q, size=len(t))]
        if N >= 3:
            uv[:, 1] = (0.0, 1.0)
            uv[:, 2] = (1.0, 0.0)
    return PairedSurfaces(name, p, q, base.ctrl, base.U, base.V, uv, knots_batched)


def config4_paired(seed: int = 41, B: int = 4096, N: int = 16384, knots_batched: bool = False):
    """The paired-points throughput workload: cfg4's nets (4096 bicubic 16x16,
    13 spans) with 16384 scattered points each = 67,108,864 points, the same count as cfg4."""
    return paired("cfg4p", B, 16, 16, 3, 3, N, seed, knots_batched)
