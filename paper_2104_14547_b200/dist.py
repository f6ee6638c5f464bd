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


def allreduce_grads(buf: GradBuffer, group=None) -> None:
    """Sum the per-rank partial gradients (fp32, NCCL over NVLink / NVSwitch on GPUs)."""
    dist.all_reduce(buf.flat, op=dist.ReduceOp.SUM, group=group)
