import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2104_14547_b200 as nb, workloads as wl, oracle
dev = torch.device('cuda')
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
for (B,n,m,p,q,nu,nv) in [(3,40,24,3,2,150,260),(1,40,24,3,2,150,260),(3,40,24,3,2,150,256),(3,12,10,3,2,150,260),(1,32,32,3,3,128,128)]:
    w = wl.surfaces("fitb", B=B, n=n, m=m, p=p, q=q, n_u=nu, n_v=nv, seed=31)
    rng = np.random.default_rng(3)
    Tf = (oracle.surface_fwd(w.ctrl, w.U, w.V, w.u, w.v, w.p, w.q) + rng.normal(0, 0.01, (B, nu, nv, 3))).astype(np.float32)
    ctrl = T(w.ctrl)
    S = nb.surface_fwd(ctrl, T(w.U), T(w.V), T(w.u), T(w.v), p, q)
    Tt = T(Tf)
    L = ((S - Tt)**2).sum().item() / (B*nu*nv)
    fitter = nb.SurfaceFitter(ctrl.clone(), T(w.U), T(w.V), T(w.u), T(w.v), Tt, p, q, 0.0)
    loss = torch.zeros(1, device=dev)
    fitter.step(loss)
    g_ref = nb.surface_bwd(ctrl, T(w.U), T(w.V), T(w.u), T(w.v), (2*(S-Tt)/(B*nu*nv)).contiguous(), p, q)
    torch.cuda.synchronize()
    print((B,n,m,p,q,nu,nv), 'loss torch', L, 'fit', loss.item(), 'grad diff', (fitter.grad - g_ref).abs().max().item(), g_ref.abs().max().item())
