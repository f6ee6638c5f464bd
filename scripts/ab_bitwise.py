"""Run the backward (and fit step) of a set of bicubic shapes through the library named by
NURBS_B200_LIB_EXPERIMENT and save the results (argv[1] = output .npz); with argv[2] = a
reference .npz, compare bitwise and print the max abs difference per case."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as wl
import paper_2104_14547_b200 as nb
dev = torch.device("cuda", 0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
cases = {
    "cfg4_64": wl.config4(B=64),
    "cfg4_batched": wl.config4(B=16, knots_batched=True),
    "cfg5_1024": wl.config5(n_u=1024, n_v=1024),
    "tiled": wl.surfaces("tl", B=2, n=120, m=24, p=3, q=3, n_u=1500, n_v=300, seed=13),
    "sparse": wl.surfaces("sp", B=2, n=60, m=40, p=3, q=3, n_u=7, n_v=5, seed=3),
    "ragged": wl.surfaces("rg", B=3, n=14, m=11, p=3, q=3, n_u=77, n_v=333, seed=14),
    "short_spans": wl.surfaces("ss", B=4, n=40, m=16, p=3, q=3, n_u=50, n_v=128, seed=15),
    "one_row": wl.surfaces("or", B=2, n=9, m=8, p=3, q=3, n_u=1, n_v=64, seed=16),
}
res = {}
for name, w in cases.items():
    g = w.grad_out(3)
    for tab in ((False,) if w.knots_batched else (False, True)):
        ctrl, U, V, u, v, gout = T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v), T(g)
        t = None
        if tab:
            sh = nb.surface_shape(ctrl, U, u, v, w.p, w.q)
            t = nb.Tables.build(sh, U, V, u, v)
        grad = nb.surface_bwd(ctrl, U, V, u, v, gout, w.p, w.q, tables=t)
        torch.cuda.synchronize()
        res[f"{name}_{int(tab)}"] = grad.cpu().numpy()
np.savez(sys.argv[1], **res)
if len(sys.argv) > 2:
    ref = np.load(sys.argv[2])
    for k in res:
        d = np.abs(res[k].astype(np.float64) - ref[k]).max()
        print(f"{k:20s} bitwise {np.array_equal(res[k], ref[k])}  max|diff| {d:.3e}")
