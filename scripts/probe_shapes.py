"""Probe: forward/backward time of the grid kernels for a few shapes (tuning experiments)."""
import sys, torch
sys.path.insert(0, '.')
import workloads as W
from paper_2104_14547_b200 import api

def run(name, B, n, m, nu, nv):
    S = W.surfaces(name, B, n, m, 3, 3, nu, nv, 7)
    dev = 'cuda'
    ctrl = torch.from_numpy(S.ctrl).to(dev); U = torch.from_numpy(S.U).to(dev); V = torch.from_numpy(S.V).to(dev)
    u = torch.from_numpy(S.u).to(dev); v = torch.from_numpy(S.v).to(dev)
    sh0 = api.surface_shape(ctrl, U, u, v, 3, 3); tab = api.Tables.build(sh0, U, V, u, v)
    out = torch.empty((B, nu, nv, 3), device=dev)
    g = torch.randn_like(out)
    gc = torch.empty_like(ctrl)
    sh = api.surface_shape(ctrl, U, u, v, 3, 3)
    ws = api.bwd_workspace_bytes(sh); wsb = torch.empty(max(ws, 1), dtype=torch.uint8, device=dev)
    def f(): api.nurbs_surface_fwd(sh, ctrl, U, V, u, v, tab, out)
    def b(): api.nurbs_surface_bwd(sh, ctrl, U, V, u, v, tab, g, gc, None, None, wsb, ws)
    res = []
    for fn in (f, b):
        for _ in range(5): fn()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(50): fn()
        e1.record(); torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 50)
    pts = B * nu * nv
    print(f"{name:28s} pts {pts/1e6:6.1f}M  fwd {res[0]*1e3:7.1f} us ({pts*12/res[0]/1e9:6.0f} GB/s)  bwd {res[1]*1e3:7.1f} us ({pts*12/res[1]/1e9:6.0f} GB/s)", flush=True)

run("cfg5 1x256x256 @8192^2", 1, 256, 256, 8192, 8192)
run("64x256x16 @8192x128", 64, 256, 16, 8192, 128)
run("512x256x16 @1024x128", 512, 256, 16, 1024, 128)
run("4x256x64 @8192x2048", 4, 256, 64, 8192, 2048)
run("16x64x256 @1024x4096", 16, 64, 256, 1024, 4096)
run("cfg4 4096x16x16 @128^2", 4096, 16, 16, 128, 128)
run("1024x16x32 @128x512", 1024, 16, 32, 128, 512)
