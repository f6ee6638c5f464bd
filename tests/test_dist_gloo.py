"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic of dist.py:
u-row sharding of one surface (config 5's partition), the flat gradient buffer the backward
writes in place, the single all-reduce (or the all-gather + rank-order sum) that combines the
partial gradients, and batch sharding of a surface batch (config 4's partition: no
collective on the data path). The per-rank results come from the fp64 oracle on that rank's
share (the CUDA path is covered by -m gpu)."""
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


def _rank_order_sum(parts, out):
    """host stand-in for nurbs_sum_partials (test only): ascending rank order"""
    acc = parts[0].clone()
    for r in range(1, parts.shape[0]):
        acc += parts[r]
    out.copy_(acc)


def _worker(rank, world, port, q, ordered=False):
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
        red = nbd.OrderedReducer(buf, sum_fn=_rank_order_sum) if ordered else None
        nbd.allreduce_grads(buf, reducer=red)
        if rank == 0:
            full = oracle.surface_bwd(w.ctrl, w.U, w.V, w.u, w.v, g, w.p, w.q)
            err = float(np.max(np.abs(buf.grad_ctrl.numpy() - full)) / np.max(np.abs(full)))
            q.put((err, float(buf.grad_U.abs().max()), float(buf.grad_V.abs().max()), buf.nbytes))
    finally:
        dist.destroy_process_group()


def _window_worker(rank, world, port, q):
    """Point sharding on the rank's sub-net (dist.row_window): each rank evaluates its u-slab
    with only the control rows / knots its spans touch, writes its partial gradient at the
    window's row offset of the full buffer, and ONE all-reduce sums the partials."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = wl.surfaces("win", B=1, n=23, m=7, p=3, q=2, n_u=61, n_v=9, seed=29)
        g = w.grad_out(8)
        a0, a1 = nbd.shard_range(w.n_u, world, rank)
        r0, r1 = nbd.row_window(w.U, w.p, w.n, float(w.u[a0]), float(w.u[a1 - 1]))
        sub_c, sub_U = w.ctrl[:, r0:r1], w.U[r0:r1 + w.p + 1]
        out = oracle.surface_fwd(sub_c, sub_U, w.V, w.u[a0:a1], w.v, w.p, w.q)
        part = oracle.surface_bwd(sub_c, sub_U, w.V, w.u[a0:a1], w.v, g[:, a0:a1], w.p, w.q)
        buf = nbd.GradBuffer.alloc(w.B, w.n, w.m, len(w.U), len(w.V), "cpu")
        buf.flat.zero_()
        buf.grad_ctrl[:, r0:r1].copy_(torch.from_numpy(part.astype(np.float32)))
        nbd.allreduce_grads(buf)
        ref_out = oracle.surface_fwd(w.ctrl, w.U, w.V, w.u[a0:a1], w.v, w.p, w.q)
        outs = [None] * world
        dist.all_gather_object(outs, (r0, r1, float(np.abs(out - ref_out).max())))
        if rank == 0:
            full = oracle.surface_bwd(w.ctrl, w.U, w.V, w.u, w.v, g, w.p, w.q)
            err = float(np.max(np.abs(buf.grad_ctrl.numpy() - full)) / np.max(np.abs(full)))
            q.put((outs, err))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_row_window_sharding_gloo():
    """The sub-net of a u-slab gives bitwise the full net's S on the slab (same spans, same
    knots in A2.2), the windows are proper sub-ranges, and the windowed partial gradients
    sum (one all-reduce) to the unsharded gradient."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_window_worker, args=(2, free_port(), q), nprocs=2, join=True)
    outs, err = q.get(timeout=60)
    assert all(e == 0.0 for _, _, e in outs)
    assert outs[0][0] == 0 and outs[-1][1] == 23 and all(r1 - r0 < 23 for r0, r1, _ in outs)
    assert err <= 1e-6


def test_row_window_edges():
    """row_window on clamped knots: samples on interior knots, at 0 and at 1, and a single
    sample; the window is [s_first-1-p, s_last+2) clamped to [0, n)."""
    U = wl.clamped_uniform_knots(10, 3)          # spans 3..9, interior knots k/7
    assert nbd.row_window(U, 3, 10, 0.0, 1.0) == (0, 10)
    assert nbd.row_window(U, 3, 10, 0.0, 0.0) == (0, 5)       # span 3 (+1) -> rows [0, 5)
    k3 = float(U[5])                                          # = 2/7: span 5 exactly on the knot
    assert nbd.row_window(U, 3, 10, k3, k3) == (1, 7)
    assert nbd.row_window(U, 3, 10, 1.0, 1.0) == (5, 10)      # span 9 (R3) -> [9-1-3, 10)
    for a, b in [(0.1, 0.2), (0.33, 0.9), (0.5, 0.5)]:
        r0, r1 = nbd.row_window(U, 3, 10, a, b)
        assert 0 <= r0 < r1 <= 10 and r1 - r0 >= 4


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
@pytest.mark.parametrize("ordered", [False, True])
def test_row_sharded_backward_allreduce_gloo(ordered):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(2, free_port(), q, ordered), nprocs=2, join=True)
    err, gU, gV, nbytes = q.get(timeout=60)
    assert err <= 1e-6          # fp32 buffer of fp64 partials, summed in one all-reduce
    assert gU == 0.0 and gV == 0.0


def _batch_worker(rank, world, port, q):
    """Config 4's partition: rank r owns surfaces shard_range(B, world, r) of ONE global batch
    and computes them with no collective; the gather below is only the test's check."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = wl.surfaces("batch", B=5, n=9, m=8, p=3, q=2, n_u=11, n_v=13, seed=23)   # odd B: ragged shards
        g = w.grad_out(6)
        b0, b1 = nbd.shard_range(w.B, world, rank)
        out = oracle.surface_fwd(w.ctrl[b0:b1], w.U, w.V, w.u, w.v, w.p, w.q)
        grad = oracle.surface_bwd(w.ctrl[b0:b1], w.U, w.V, w.u, w.v, g[b0:b1], w.p, w.q)
        counts = [None] * world
        dist.all_gather_object(counts, (b0, b1, out, grad))
        if rank == 0:
            assert [c[0] for c in counts] == [0, 3] and [c[1] for c in counts] == [3, 5]
            full_out = np.concatenate([c[2] for c in counts])
            full_grad = np.concatenate([c[3] for c in counts])
            ref_out = oracle.surface_fwd(w.ctrl, w.U, w.V, w.u, w.v, w.p, w.q)
            ref_grad = oracle.surface_bwd(w.ctrl, w.U, w.V, w.u, w.v, g, w.p, w.q)
            q.put((full_out.shape[0], float(np.abs(full_out - ref_out).max()), float(np.abs(full_grad - ref_grad).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_batch_sharded_surfaces_gloo():
    """Strong batch sharding: the ranks' shards tile the ONE global batch (no surface twice,
    none missing) and, surfaces being independent (Alg.1), the shard results are
    exactly the unsharded ones."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_batch_worker, args=(2, free_port(), q), nprocs=2, join=True)
    B, e_out, e_grad = q.get(timeout=60)
    assert B == 5 and e_out == 0.0 and e_grad == 0.0


def test_pin_nccl_order_keeps_caller_settings(monkeypatch):
    monkeypatch.delenv("NCCL_ALGO", raising=False)
    monkeypatch.setenv("NCCL_PROTO", "LL128")
    assert nbd.pin_nccl_order() == {"NCCL_ALGO": "Ring", "NCCL_PROTO": "LL128"}


def test_init_nccl_sets_failure_detection(monkeypatch):
    """init_nccl turns on NCCL's asynchronous error handling, pins the reduction order and
    passes a collective timeout (the process-group call itself is stubbed: no GPU here)."""
    import datetime
    calls = {}
    monkeypatch.delenv("TORCH_NCCL_ASYNC_ERROR_HANDLING", raising=False)
    monkeypatch.delenv("NCCL_ALGO", raising=False)
    monkeypatch.delenv("NCCL_PROTO", raising=False)
    monkeypatch.setattr(nbd.dist, "init_process_group", lambda backend, **kw: calls.update(backend=backend, **kw))
    nbd.init_nccl("cuda:0", timeout_s=30.0)
    assert calls["backend"] == "nccl" and calls["timeout"] == datetime.timedelta(seconds=30)
    assert os.environ["TORCH_NCCL_ASYNC_ERROR_HANDLING"] == "1"
    assert os.environ["NCCL_ALGO"] == "Ring" and os.environ["NCCL_PROTO"] == "Simple"
