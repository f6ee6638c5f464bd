import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2104_14547_b200 as nb, workloads as wl, oracle
dev = torch.device('cuda')
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
B,n,m,p,q,nu,nv = 3,12,10,3,3,150,260
w = wl.surfaces("fitb", B=B, n=n, m=m, p=p, q=q, n_u=nu, n_v=nv, seed=31)
Tf = oracle.surface_fwd(w.ctrl, w.U, w.V, w.u, w.v, w.p, w.q).astype(np.float32)
ctrl = T(w.ctrl); Tt = T(Tf)
fitter = nb.SurfaceFitter(ctrl.clone(), T(w.U), T(w.V), T(w.u), T(w.v), Tt, p, q, 0.0)
fitter.ws.fill_(7)
loss = torch.zeros(1, device=dev)
fitter.step(loss); torch.cuda.synchronize()
wsb = nb.bwd_workspace_bytes(fitter.sh)
parts = fitter.ws[wsb:].view(torch.float32).cpu().numpy()
print('ws', wsb, fitter.ws_bytes, 'parts', parts[:40])
import ctypes
