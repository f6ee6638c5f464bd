"""Cases run under compute-sanitizer (memcheck / racecheck / synccheck), one process per tool:
config 1 (curve), config 2, a tiled config-5 net on a 1024^2 grid (reduce path, tensor-map IO),
the per-thread IO path, paired points (fwd + bwd), the fused fit step, the knot-gradient
backward, the derivatives, and unsorted samples in unchecked mode (memory safety).
Usage: python scripts/sanitize_cases.py [case ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_14547_b200 as nb  # noqa: E402
import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731


def surf(w, tables=False, u=None, v=None):
    u = w.u if u is None else u
    v = w.v if v is None else v
    ctrl, U, V, uu, vv = T(w.ctrl), T(w.U), T(w.V), T(u), T(v)
    tab = nb.Tables.build(nb.surface_shape(ctrl, U, uu, vv, w.p, w.q), U, V, uu, vv) if tables else None
    out = nb.surface_fwd(ctrl, U, V, uu, vv, w.p, w.q, tables=tab)
    nb.surface_bwd(ctrl, U, V, uu, vv, torch.ones_like(out), w.p, w.q, tables=tab,
                   grad_U=torch.empty_like(U), grad_V=torch.empty_like(V))


def case_cfg1():
    c = wl.config1()
    out = nb.curve_fwd(T(c.ctrl), T(c.U), T(c.u), c.p)
    nb.curve_bwd(T(c.ctrl), T(c.U), T(c.u), torch.ones_like(out), c.p)


def case_cfg2():
    surf(wl.config2(), tables=True)


def case_cfg5_tiled():
    surf(wl.config5(n_u=1024, n_v=1024), tables=True)


def case_direct_io():
    surf(wl.surfaces("dio", B=2, n=11, m=9, p=3, q=3, n_u=45, n_v=130, seed=1))


def case_paired():
    w = wl.paired("sp", B=3, n=16, m=16, p=3, q=3, N=5000, seed=2)
    ctrl, U, V, uv = T(w.ctrl), T(w.U), T(w.V), T(w.uv)
    out = nb.surface_points_fwd(ctrl, U, V, uv, 3, 3)
    nb.surface_points_bwd(ctrl, U, V, uv, torch.ones_like(out), 3, 3)


def case_fit():
    truth, init = wl.config3_fit(n_s=128)
    U, V, u, v = T(truth.U), T(truth.V), T(truth.u), T(truth.v)
    target = nb.surface_fwd(T(truth.ctrl), U, V, u, v, 3, 3)
    f = nb.SurfaceFitter(T(init.ctrl), U, V, u, v, target, 3, 3, lr=100.0)
    f.run(3, graph=False)


def case_knots():
    w = wl.config5(n_u=600, n_v=400)
    ctrl, U, V, u, v = T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v)
    nb.surface_bwd_knots(ctrl, U, V, u, v, torch.ones((1, 600, 400, 3), device=dev), 3, 3)


def case_derivs():
    w = wl.config4(B=4)
    nb.surface_derivs(T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v), 3, 3)


def case_unsorted():
    rng = np.random.default_rng(1)
    for w in (wl.config4(B=2), wl.config5(n_u=400, n_v=300)):
        surf(w, u=w.u[rng.permutation(w.n_u)].copy(), v=w.v[::-1].copy())


def case_shard_plans():
    """the round-2 plans: config 4 below kDirectMinB (tiled + reduce) and a config-5 u-slab on
    its sub-net window (dist.row_window)"""
    surf(wl.config4(B=20), tables=True)
    from paper_2104_14547_b200 import dist as nbd
    w = wl.config5(n_u=512, n_v=256)
    a0, a1 = nbd.shard_range(w.n_u, 8, 3)
    r0, r1 = nbd.row_window(w.U, w.p, w.n, float(w.u[a0]), float(w.u[a1 - 1]))
    surf(wl.Surfaces(name="win", p=w.p, q=w.q, ctrl=w.ctrl[:, r0:r1].copy(), U=w.U[r0:r1 + w.p + 1].copy(),
                     V=w.V, u=w.u[a0:a1].copy(), v=w.v), tables=True)


CASES = {k[5:]: f for k, f in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        torch.cuda.synchronize()
        print("case ok:", name, flush=True)
