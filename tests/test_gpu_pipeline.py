"""GPU: HostBatchPipeline (host-resident batches, PCIe copies overlapped with the kernels)
returns exactly what the device calls return, on a ragged chunking, and against the oracle."""
import numpy as np
import pytest

import oracle
import workloads as wl

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_14547_b200 as nb  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2104_14547_b200.build import build
    build()
    oracle.build()


@pytest.mark.parametrize("chunk,use_tables", [(8, True), (37, False), (5, True)])
def test_pipeline_equals_device_calls(chunk, use_tables):
    w = wl.surfaces("pipe", 37, 16, 16, 3, 3, 128, 128, seed=91)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    ctrl, U, V, u, v = T(w.ctrl), T(w.U), T(w.V), T(w.u), T(w.v)
    rng = np.random.default_rng(92)
    g = rng.standard_normal((w.B, w.n_u, w.n_v, 3)).astype(np.float32)
    sh = nb.nurbs_shape(w.B, w.n, w.m, w.p, w.q, w.n_u, w.n_v, 0)
    tables = nb.Tables.build(sh, U, V, u, v) if use_tables else None
    # reference: the device calls on the same chunks (a chunk's plan, hence its summation
    # order, is a function of its shape) -> bitwise; the whole batch in one call -> R16
    ref_out = torch.cat([nb.surface_fwd(ctrl[b:b + chunk], U, V, u, v, 3, 3, tables=tables)
                         for b in range(0, w.B, chunk)])
    ref_grad = torch.cat([nb.surface_bwd(ctrl[b:b + chunk], U, V, u, v, T(g[b:b + chunk]), 3, 3, tables=tables)
                          for b in range(0, w.B, chunk)])
    whole = nb.surface_bwd(ctrl, U, V, u, v, T(g), 3, 3, tables=tables)
    assert float((whole - ref_grad).abs().max() / whole.abs().max()) <= 1e-4

    pipe = nb.HostBatchPipeline(w.n, w.m, 3, 3, U, V, u, v, tables, chunk=chunk, device=DEV)
    h_ctrl = torch.from_numpy(w.ctrl.copy()).pin_memory()
    h_gout = torch.from_numpy(g).pin_memory()
    h_out = torch.empty((w.B, w.n_u, w.n_v, 3)).pin_memory()
    h_grad = torch.empty((w.B, w.n, w.m, 4)).pin_memory()
    for _ in range(2):  # a second call reuses the slots (event chain across calls)
        h_out.zero_(); h_grad.zero_()
        pipe.fwd_bwd(h_ctrl, h_gout, h_out, h_grad)
        torch.cuda.synchronize()
        assert torch.equal(h_out, ref_out.cpu())
        assert torch.equal(h_grad, ref_grad.cpu())
    assert pipe.h2d_bytes(w.B) == w.B * (16 * 16 * 16 + 128 * 128 * 12)

    # and one surface against the fp64 oracle (forward, normwise R16)
    k = 20
    S = oracle.surface_fwd(w.ctrl[k:k + 1], w.U, w.V, w.u, w.v, 3, 3)
    err = np.abs(h_out[k].numpy() - S[0]).max() / np.abs(w.ctrl[k, ..., :3]).max()
    assert err <= 1e-5


def test_pipeline_rejects_bad_buffers():
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    with pytest.raises(ValueError):
        nb.HostBatchPipeline(16, 16, 3, 3, T(np.zeros(20, np.float32)), None, T(np.zeros(4, np.float32)),
                             T(np.zeros(4, np.float32)), None, chunk=0, device=DEV)
    w = wl.surfaces("pipe3", 2, 16, 16, 3, 3, 64, 64, seed=94)
    U, V, u, v = T(w.U), T(w.V), T(w.u), T(w.v)
    pipe = nb.HostBatchPipeline(16, 16, 3, 3, U, V, u, v, None, chunk=1, device=DEV)
    bad = torch.empty((2, 64, 64, 3), device=DEV)
    with pytest.raises(ValueError):
        pipe.fwd_bwd(torch.zeros(2, 16, 16, 4), torch.zeros(2, 64, 64, 3), bad, torch.zeros(2, 16, 16, 4))
