"""Multi-GPU partitioning of the hot path, one process per GPU.

* Batch sharding (config 4): surfaces are independent units (Alg.1 "for k = 1: surfaces in
  parallel") — each rank owns whole surfaces; there is no data-path collective.
* Point sharding of one surface (config 5): rank r owns a contiguous slab of u-rows
  [a0, a1) of the parameter grid (its `out` / `grad_out` rows are one contiguous slab and
  its samples are u[a0:a1]). The forward needs no communication; the backward produces
  partial gradients that are summed by ONE all-reduce of a packed buffer
  [dP,dw (B*n*m*4) | dU | dV] (the knot parts are zero by definition, but are part of
  the Psi-gradient the paper returns, so they travel in the same buffer).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def row_window(U, p: int, n: int, u_first: float, u_last: float) -> tuple[int, int]:
    """Control rows [r0, r1) that the samples u in [u_first, u_last] (sorted) can touch.

    Local support (only p+1 basis functions are non-zero at u, those of span s cover
    control rows s-p..s): a rank that owns the u-rows of a slab needs only the control rows
    of the knot spans its samples fall in. Passing the sub-net ctrl[:, r0:r1] with the knot
    slice U[r0 : r1+p+1] (a valid knot vector of n' = r1-r0 control points whose domain
    [U[r0+p], U[r1]] contains the slab) gives every sample the same span (shifted by r0) and
    the same knots in A2.2, hence bitwise the same S and the same partial gradient rows
    (written at row offset r0 of the full gradient). Host logic only: the span of a sample is
    the largest s with U[s] <= u, clamped to [p, n-1]; the window is widened by one span on
    each side, so a sample on a knot or at the domain end is covered whatever tie rule
    FindSpan uses (R3/R4). Returns (r0, r1)."""
    import numpy as np
    Uh = np.asarray(U, dtype=np.float32)
    s = np.searchsorted(Uh, np.array([u_first, u_last], dtype=np.float32), side="right") - 1
    sa = int(min(max(s[0], p), n - 1))
    sb = int(min(max(s[1], p), n - 1))
    sa, sb = max(p, sa - 1), min(n - 1, sb + 1)
    return sa - p, sb + 1


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced split of [0, total) (first `total % world` ranks get one more)."""
    base, extra = divmod(total, world)
    a0 = rank * base + min(rank, extra)
    return a0, a0 + base + (1 if rank < extra else 0)


@dataclass
class GradBuffer:
    """One flat fp32 buffer viewed as grad_ctrl [B][n][m][4], grad_U, grad_V — the backward
    writes into the views and the all-reduce runs on `flat` (no packing copy)."""
    flat: torch.Tensor
    grad_ctrl: torch.Tensor
    grad_U: torch.Tensor
    grad_V: torch.Tensor

    @staticmethod
    def alloc(B: int, n: int, m: int, len_U: int, len_V: int, device) -> "GradBuffer":
        nc = B * n * m * 4
        flat = torch.empty(nc + len_U + len_V, dtype=torch.float32, device=device)
        return GradBuffer(flat, flat[:nc].view(B, n, m, 4), flat[nc:nc + len_U], flat[nc + len_U:])

    @property
    def nbytes(self) -> int:
        return self.flat.numel() * 4


# NCCL settings that fix the all-reduce's summation order for a given world size and
# topology (one algorithm, one protocol); set before the process group is created. With
# `ordered=True` the order is fixed by construction instead (all-gather + rank-order sum).
NCCL_DETERMINISTIC_ENV = {"NCCL_ALGO": "Ring", "NCCL_PROTO": "Simple"}


def pin_nccl_order() -> dict:
    """Set NCCL_ALGO / NCCL_PROTO (unless the caller already did); returns what is in effect."""
    import os
    for k, v in NCCL_DETERMINISTIC_ENV.items():
        os.environ.setdefault(k, v)
    return {k: os.environ[k] for k in NCCL_DETERMINISTIC_ENV}


class OrderedReducer:
    """All-gather of the per-rank partials into [world][N], then ONE fixed-order sum
    (ascending rank) in the library's nurbs_sum_partials kernel: bitwise repeatable for a
    given world size whatever NCCL's algorithm. Costs an all-gather of world x N floats (8 MB
    for config 5 at G = 8) instead of an all-reduce of N."""

    def __init__(self, buf: GradBuffer, group=None, sum_fn=None):
        self.world = dist.get_world_size(group)
        self.group = group
        self.gathered = torch.empty(self.world * buf.flat.numel(), dtype=buf.flat.dtype, device=buf.flat.device)
        if sum_fn is None:
            if not buf.flat.is_cuda:
                raise RuntimeError("OrderedReducer sums on the GPU (nurbs_sum_partials); pass sum_fn for host tensors")
            from .api import nurbs_sum_partials
            sum_fn = nurbs_sum_partials
        self.sum_fn = sum_fn

    def __call__(self, buf: GradBuffer) -> None:
        dist.all_gather_into_tensor(self.gathered, buf.flat, group=self.group)
        self.sum_fn(self.gathered.view(self.world, -1), buf.flat)


def init_nccl(device, timeout_s: float = 120.0) -> None:
    """One process per GPU over NCCL with failure detection: NCCL's asynchronous error handling
    on (a rank that hits a communicator error or a collective that exceeds `timeout_s` aborts
    the process group and raises instead of hanging the job), order pinned for the gradient
    all-reduce (pin_nccl_order). Call once per rank; RANK / WORLD_SIZE / MASTER_* from the
    environment (torch.distributed.run)."""
    import datetime
    import os
    os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
    pin_nccl_order()
    dist.init_process_group("nccl", device_id=device, timeout=datetime.timedelta(seconds=timeout_s))


def allreduce_grads(buf: GradBuffer, group=None, reducer: "OrderedReducer | None" = None) -> None:
    """Sum the per-rank partial gradients: one NCCL all-reduce over NVLink / NVSwitch (order
    fixed by pin_nccl_order), or, with an OrderedReducer, all-gather + rank-order sum."""
    if reducer is not None:
        reducer(buf)
    else:
        dist.all_reduce(buf.flat, op=dist.ReduceOp.SUM, group=group)
