"""GPU: seeded random shapes through every IO path of the grid kernels (per-thread, TMA bulk,
2-D tensor map; one tile or several; tables or in-kernel bases; shared or per-surface knots),
forward and backward against the fp64 oracle (normwise R16 tolerances), and the knot
gradients of the same call zero-filled."""
import numpy as np
import pytest

import workloads as wl

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from test_gpu_parity import check_surface  # noqa: E402


def _case(seed):
    rng = np.random.default_rng(9000 + seed)
    p, q = int(rng.integers(1, 6)), int(rng.integers(1, 6))
    n, m = int(rng.integers(p + 1, 24)), int(rng.integers(q + 1, 40))
    B = int(rng.integers(1, 5))
    n_u = int(rng.integers(1, 260))
    # mostly multiples of 4 (TMA paths), some ragged (per-thread path)
    n_v = int(rng.choice([4, 60, 64, 68, 128, 132, 192, 256, 300, 388, 7, 45, 131]))
    batched = bool(rng.integers(0, 2))
    tables = bool(rng.integers(0, 2)) and not batched
    return p, q, n, m, B, n_u, n_v, batched, tables


@pytest.mark.parametrize("seed", range(64))
def test_random_shapes(seed):
    p, q, n, m, B, n_u, n_v, batched, tables = _case(seed)
    w = wl.surfaces(f"fuzz{seed}", B=B, n=n, m=m, p=p, q=q, n_u=n_u, n_v=n_v, seed=seed, knots_batched=batched)
    check_surface(w, gseed=seed, tables=tables)
