"""Probe: config 4 fwd+bwd, whole batch sequentially vs chunks whose backward overlaps the next
chunk's forward on a second stream (tuning experiment; not the bench)."""
import sys, torch
sys.path.insert(0, '.')
import workloads as W
import paper_2104_14547_b200 as nb

w = W.config4()
dev = 'cuda'
T = lambda a: torch.from_numpy(a.copy()).to(dev)
ctrl, U, V, u, v = T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v)
B = w.B
out = torch.empty((B, 128, 128, 3), device=dev)
g = torch.randn_like(out)
gc = torch.empty_like(ctrl)
sh_full = nb.nurbs_shape(B, 16, 16, 3, 3, 128, 128, 0)
tab = nb.Tables.build(sh_full, U, V, u, v)

def run(C):
    shc = nb.nurbs_shape(B // C, 16, 16, 3, 3, 128, 128, 0)
    ws = nb.bwd_workspace_bytes(shc)
    wsb = [torch.empty(max(ws, 1), dtype=torch.uint8, device=dev) for _ in range(C)]
    s1, s2 = torch.cuda.current_stream(), torch.cuda.Stream()
    evs = [torch.cuda.Event() for _ in range(C)]
    def step():
        for k in range(C):
            sl = slice(k * B // C, (k + 1) * B // C)
            nb.nurbs_surface_fwd(shc, ctrl[sl], U, V, u, v, tab, out[sl], s1)
            evs[k].record(s1)
            s2.wait_event(evs[k])
            nb.nurbs_surface_bwd(shc, ctrl[sl], U, V, u, v, tab, g[sl], gc[sl], None, None, wsb[k], ws, s2)
        e = torch.cuda.Event(); e.record(s2); s1.wait_event(e)
    for _ in range(5): step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(s1)
    for _ in range(50): step()
    e1.record(s1); torch.cuda.synchronize()
    print(f"chunks {C}: {e0.elapsed_time(e1)/50*1e3:.1f} us per step (ws {ws})", flush=True)

for C in (1, 2, 4, 8):
    run(C)
