"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic of dist.py:
u-row sharding of one surface (config 5's partition), the flat gradient buffer the backward
writes in place, and the single all-reduce that combines the partial gradients. The per-rank
partials come from the fp64 oracle on that rank's rows (the CUDA path is covered by -m gpu)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as wl
from paper_2104_14547_b200 import dist as nbd


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = wl.surfaces("dist", B=1, n=12, m=9, p=3, q=2, n_u=37, n_v=29, seed=21)
        g = w.grad_out(5)
        a0, a1 = nbd.shard_range(w.n_u, world, rank)
        buf = nbd.GradBuffer.alloc(w.B, w.n, w.m, len(w.U), len(w.V), "cpu")
        part = oracle.surface_bwd(w.ctrl, w.U, w.V, w.u[a0:a1], w.v, g[:, a0:a1], w.p, w.q)
        buf.grad_ctrl.copy_(torch.from_numpy(part.astype(np.float32)))
        buf.grad_U.fill_(0.0)   # the library zero-fills knot gradients
        buf.grad_V.fill_(0.0)
        nbd.allreduce_grads(buf)
        if rank == 0:
            full = oracle.surface_bwd(w.ctrl, w.U, w.V, w.u, w.v, g, w.p, w.q)
            err = float(np.max(np.abs(buf.grad_ctrl.numpy() - full)) / np.max(np.abs(full)))
            q.put((err, float(buf.grad_U.abs().max()), float(buf.grad_V.abs().max()), buf.nbytes))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for total in (0, 1, 7, 8192, 8191):
        for world in (1, 2, 3, 8):
            ranges = [nbd.shard_range(total, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_gradbuffer_views_share_storage():
    buf = nbd.GradBuffer.alloc(2, 3, 4, 7, 8, "cpu")
    buf.flat.zero_()
    buf.grad_ctrl[1, 2, 3, 3] = 5.0
    buf.grad_V[-1] = 2.0
    assert buf.flat[2 * 3 * 4 * 4 - 1] == 5.0 and buf.flat[-1] == 2.0
    assert buf.nbytes == (2 * 3 * 4 * 4 + 15) * 4
    # config 5: [dP,dw | dU | dV] = 256*256*4 + 260 + 260 floats = 1,050,656 B
    assert (256 * 256 * 4 + 260 + 260) * 4 == 1050656


@pytest.mark.timeout(180)
def test_row_sharded_backward_allreduce_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(2, free_port(), q), nprocs=2, join=True)
    err, gU, gV, nbytes = q.get(timeout=60)
    assert err <= 1e-6          # fp32 buffer of fp64 partials, summed in one all-reduce
    assert gU == 0.0 and gV == 0.0
