"""Host-resident batches: the surface forward + backward of a batch that lives in (pinned)
host memory, with the PCIe copies overlapped with the kernels.

The library calls (include/nurbs.h) take device pointers. A caller whose control nets and
upstream gradients dL/dS are in host memory must copy them over PCIe, and that copy — not
the kernels — bounds the end-to-end rate (config 4: 822 MB in and 822 MB out per step
against ~0.35 ms of kernels). ``HostBatchPipeline`` splits the batch into chunks of whole
surfaces (surfaces are independent units, Alg.1) and runs three CUDA streams:

    h2d stream:      ctrl[k], grad_out[k]  host -> device      (copy engine 0)
    compute stream:  nurbs_surface_fwd + nurbs_surface_bwd on chunk k
    d2h stream:      out[k], grad_ctrl[k]  device -> host      (copy engine 1)

with two device slots, so chunk k+1 uploads and chunk k-1 downloads while chunk k
computes; the two copy directions run concurrently. This is plumbing only (device memory,
streams, events): every arithmetic step runs in libnurbs_b200.so, through the same C-ABI
calls as ``api.nurbs_surface_fwd`` / ``api.nurbs_surface_bwd``.
"""
from __future__ import annotations

import torch

from . import api
from ._abi import nurbs_shape


class HostBatchPipeline:
    """Forward + backward of a host-resident batch of surfaces on one device.

    Shapes follow include/nurbs.h: ``ctrl[B][n][m][4]``, ``grad_out`` and ``out``
    ``[B][n_u][n_v][3]``, ``grad_ctrl[B][n][m][4]`` (overwritten); knots, parameters and the
    optional tables are device tensors shared by the whole batch (``knots_batched = 0``).
    The knot gradients are zero by definition and are not produced here.
    """

    def __init__(self, n: int, m: int, p: int, q: int, U, V, u, v, tables=None, chunk: int = 256,
                 device=None):
        self.device = torch.device(device if device is not None else U.device)
        self.n, self.m, self.p, self.q = n, m, p, q
        self.U, self.V, self.u, self.v, self.tables = U, V, u, v, tables
        self.n_u, self.n_v = u.numel(), v.numel()
        self.chunk = int(chunk)
        if self.chunk < 1:
            raise ValueError("chunk must be >= 1 surface")
        C, dev = self.chunk, self.device
        self.sh = nurbs_shape(C, n, m, p, q, self.n_u, self.n_v, 0)
        f32 = torch.float32
        self.d_ctrl = [torch.empty((C, n, m, 4), dtype=f32, device=dev) for _ in range(2)]
        self.d_gout = [torch.empty((C, self.n_u, self.n_v, 3), dtype=f32, device=dev) for _ in range(2)]
        self.d_out = [torch.empty((C, self.n_u, self.n_v, 3), dtype=f32, device=dev) for _ in range(2)]
        self.d_grad = [torch.empty((C, n, m, 4), dtype=f32, device=dev) for _ in range(2)]
        # backward workspace per slot (a chunk may be planned as several tiles per surface);
        # sized for every chunk length up to C (the plan is a pure function of the shape)
        self.ws_cap = max(api.bwd_workspace_bytes(nurbs_shape(b, n, m, p, q, self.n_u, self.n_v, 0))
                          for b in range(1, C + 1))
        self.d_ws = [torch.empty(max(self.ws_cap, 1), dtype=torch.uint8, device=dev) for _ in range(2)]
        self.s_h2d = torch.cuda.Stream(dev)
        self.s_comp = torch.cuda.Stream(dev)
        self.s_d2h = torch.cuda.Stream(dev)
        ev = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
        self.e_up, self.e_comp, self.e_down = ev(), ev(), ev()
        self._used = [False, False]

    def h2d_bytes(self, B: int) -> int:
        return B * (self.n * self.m * 16 + self.n_u * self.n_v * 12)

    def d2h_bytes(self, B: int) -> int:
        return B * (self.n * self.m * 16 + self.n_u * self.n_v * 12)

    def fwd_bwd(self, h_ctrl, h_gout, h_out, h_grad, stream=None):
        """Enqueue S = fwd(ctrl) into ``h_out`` and dL/d(P, w) into ``h_grad`` for the whole
        host batch. Host tensors should be pinned (pageable memory serialises the copies).
        Asynchronous: the work is ordered after ``stream`` (default: the current stream) and
        ``stream`` waits for its completion, so an event recorded on it afterwards (or a
        synchronize) covers the whole batch."""
        B = h_ctrl.shape[0]
        for t, shp in ((h_gout, (B, self.n_u, self.n_v, 3)), (h_out, (B, self.n_u, self.n_v, 3)),
                       (h_grad, (B, self.n, self.m, 4)), (h_ctrl, (B, self.n, self.m, 4))):
            if tuple(t.shape) != shp or t.is_cuda or not t.is_contiguous():
                raise ValueError(f"expected a contiguous host tensor of shape {shp}, got {tuple(t.shape)}")
        caller = stream if stream is not None else torch.cuda.current_stream(self.device)
        start = torch.cuda.Event()
        start.record(caller)
        for s in (self.s_h2d, self.s_comp, self.s_d2h):
            s.wait_event(start)
        C = self.chunk
        for k, b0 in enumerate(range(0, B, C)):
            b1 = min(B, b0 + C)
            nb = b1 - b0
            sl = k & 1
            # upload chunk k into slot sl once the chunk that last used the slot has computed
            if self._used[sl]:
                self.s_h2d.wait_event(self.e_comp[sl])
            with torch.cuda.stream(self.s_h2d):
                self.d_ctrl[sl][:nb].copy_(h_ctrl[b0:b1], non_blocking=True)
                self.d_gout[sl][:nb].copy_(h_gout[b0:b1], non_blocking=True)
            self.e_up[sl].record(self.s_h2d)
            # compute once uploaded and once the slot's previous outputs have been downloaded
            self.s_comp.wait_event(self.e_up[sl])
            if self._used[sl]:
                self.s_comp.wait_event(self.e_down[sl])
            sh = self.sh if nb == C else nurbs_shape(nb, self.n, self.m, self.p, self.q, self.n_u, self.n_v, 0)
            api.nurbs_surface_fwd(sh, self.d_ctrl[sl], self.U, self.V, self.u, self.v, self.tables,
                                  self.d_out[sl], self.s_comp)
            ws = api.bwd_workspace_bytes(sh)
            api.nurbs_surface_bwd(sh, self.d_ctrl[sl], self.U, self.V, self.u, self.v, self.tables,
                                  self.d_gout[sl], self.d_grad[sl], None, None, self.d_ws[sl], ws, self.s_comp)
            self.e_comp[sl].record(self.s_comp)
            # download the results
            self.s_d2h.wait_event(self.e_comp[sl])
            with torch.cuda.stream(self.s_d2h):
                h_out[b0:b1].copy_(self.d_out[sl][:nb], non_blocking=True)
                h_grad[b0:b1].copy_(self.d_grad[sl][:nb], non_blocking=True)
            self.e_down[sl].record(self.s_d2h)
            self._used[sl] = True
        done = torch.cuda.Event()
        done.record(self.s_d2h)
        caller.wait_event(done)
        # the compute and h2d streams finished before the last download (event chain)
