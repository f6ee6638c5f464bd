"""CPU checks of the boundary: the C-ABI library builds for sm_100a, loads without a GPU,
exports every symbol include/nurbs.h declares, and its host-only entry points behave
(no kernel launches here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2104_14547_b200.build import build
    build()
    from paper_2104_14547_b200 import _abi
    return _abi.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "nurbs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nurbs_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(lib):
    from paper_2104_14547_b200 import _abi
    decl = declared_symbols()
    assert sorted(_abi.EXPORTS) == decl
    nm = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (nurbs_[a-z0-9_]+)$", nm, flags=re.M))
    assert set(decl) <= exported, set(decl) - exported
    for name in decl:
        getattr(lib, name)


def test_sass_is_sm100a(lib):
    from paper_2104_14547_b200 import _abi
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass            # TMA bulk copies (cp.async.bulk) in the grid kernels
    assert "SYNCS" in sass             # mbarrier pipeline


def test_host_only_entry_points(lib):
    from paper_2104_14547_b200 import _abi
    assert lib.nurbs_abi_version() == 1
    assert lib.nurbs_strerror(0) == b"ok"
    assert lib.nurbs_strerror(8) == b"workspace missing or too small"
    sh = _abi.nurbs_shape(4096, 16, 16, 3, 3, 128, 128, 0)
    assert lib.nurbs_surface_bwd_workspace_bytes(ctypes.byref(sh)) == 0      # one tile per surface
    big = _abi.nurbs_shape(1, 256, 256, 3, 3, 8192, 8192, 0)
    assert lib.nurbs_surface_bwd_workspace_bytes(ctypes.byref(big)) > 0       # cross-tile reduction
    assert lib.nurbs_tables_bytes(ctypes.byref(sh)) >= 256 + 128 * 4 * 2 + 128 * 4 * 4 * 2
    curve = _abi.nurbs_shape(1, 6, 1, 3, 0, 100, 1, 0)
    assert lib.nurbs_curve_bwd_workspace_bytes(ctypes.byref(curve)) == 0


def test_shape_errors_need_no_gpu(lib):
    from paper_2104_14547_b200 import _abi
    P = None
    bad_deg = _abi.nurbs_shape(1, 8, 8, 6, 3, 4, 4, 0)
    st = lib.nurbs_surface_fwd(ctypes.byref(bad_deg), 16, 16, 16, 16, 16, P, 16, P)
    assert st == 2 and b"degree" in lib.nurbs_last_error_detail()
    few = _abi.nurbs_shape(1, 3, 8, 3, 3, 4, 4, 0)
    assert lib.nurbs_surface_fwd(ctypes.byref(few), 16, 16, 16, 16, 16, P, 16, P) == 1
    assert lib.nurbs_surface_fwd(None, 16, 16, 16, 16, 16, P, 16, P) == 1
    sh = _abi.nurbs_shape(1, 8, 8, 3, 3, 4, 4, 0)
    assert lib.nurbs_surface_fwd(ctypes.byref(sh), None, 16, 16, 16, 16, P, 16, P) == 1   # NULL ctrl
    assert lib.nurbs_surface_fwd(ctypes.byref(sh), 20, 16, 16, 16, 16, P, 16, P) == 1     # misaligned
    notcurve = _abi.nurbs_shape(1, 6, 2, 3, 0, 10, 1, 0)
    assert lib.nurbs_curve_fwd(ctypes.byref(notcurve), 16, 16, 16, P, 16, P) == 1
    batched = _abi.nurbs_shape(2, 8, 8, 3, 3, 4, 4, 1)
    assert lib.nurbs_surface_fwd(ctypes.byref(batched), 16, 16, 16, 16, 16, 32, 16, P) == 9  # tables+batched


def test_plan_is_bounded(lib):
    """The library's own plan (nurbs_grid_plan): row-block bands never exceed the kRMax = 16
    staged control rows, the row blocks cover every knot span, the column blocks every
    sample, one tile per surface means no workspace, and the plan is a function of the shape
    alone (asked twice, same answer)."""
    import math
    from paper_2104_14547_b200 import _abi, api
    for (B, n, p, n_u, m, n_v) in [(4096, 16, 3, 128, 16, 128), (512, 16, 3, 128, 16, 128), (1, 256, 3, 8192, 256, 8192),
                                   (1, 256, 3, 1024, 256, 8192), (1, 8, 3, 64, 8, 64), (1, 32, 3, 512, 32, 512),
                                   (7, 40, 5, 9, 11, 300), (1, 6, 3, 100, 6, 100)]:
        sh = _abi.nurbs_shape(B, n, m, p, 3 if m > 3 else 1, n_u, n_v, 0)
        pl = api.grid_plan(sh)
        assert pl == api.grid_plan(sh)
        spans = n - p
        assert pl["K"] + p <= 16 or n <= 16
        assert pl["row_blocks"] * pl["K"] >= spans and (pl["row_blocks"] - 1) * pl["K"] < spans
        assert pl["col_blocks"] == math.ceil(n_v / 128)
        assert pl["band_rows"] == min(pl["K"] + p, n)
        assert pl["ctas"] == B * pl["row_blocks"] * pl["col_blocks"]
        ws = lib.nurbs_surface_bwd_workspace_bytes(ctypes.byref(sh))
        assert (ws == 0) == bool(pl["direct"]) and pl["direct"] == (pl["ctas"] == B)
    # config 4 keeps one CTA per surface (no reduction); config 5 is tiled
    assert api.grid_plan(_abi.nurbs_shape(4096, 16, 16, 3, 3, 128, 128, 0))["direct"] == 1
    assert api.grid_plan(_abi.nurbs_shape(1, 256, 256, 3, 3, 8192, 8192, 0))["direct"] == 0
    curve = api.grid_plan(_abi.nurbs_shape(1, 6, 1, 3, 0, 100, 1, 0))
    assert curve["row_blocks"] == 1 and curve["col_blocks"] == 1
    assert lib.nurbs_grid_plan(None, (ctypes.c_int32 * 6)()) == 1


def test_plan_rules_at_the_measured_shapes(lib):
    """The backward plan's fitted rules (profiles/r02_plan_sweep.txt) at the shapes
    they were fitted on: one tile per surface for config 4 from B = 128 surfaces up (every
    per-rank shard of the 1..8-GPU runs), tiled below; config 5 and its sub-net windows take
    the sweep's best K (7, and 4 for the 8-way window)."""
    from paper_2104_14547_b200 import _abi, api
    cfg4 = lambda B: api.grid_plan(_abi.nurbs_shape(B, 16, 16, 3, 3, 128, 128, 0))  # noqa: E731
    for B in (4096, 2048, 1024, 512, 128):
        assert cfg4(B)["direct"] == 1 and cfg4(B)["K"] == 13
    assert cfg4(127)["direct"] == 0 and cfg4(1)["direct"] == 0
    assert api.grid_plan(_abi.nurbs_shape(1, 256, 256, 3, 3, 8192, 8192, 0))["K"] == 7
    assert api.grid_plan(_abi.nurbs_shape(1, 131, 256, 3, 3, 4096, 8192, 0))["K"] == 7    # G = 2 window
    assert api.grid_plan(_abi.nurbs_shape(1, 68, 256, 3, 3, 2048, 8192, 0))["K"] == 7     # G = 4
    assert api.grid_plan(_abi.nurbs_shape(1, 36, 256, 3, 3, 1024, 8192, 0))["K"] == 4     # G = 8
    # configs 2 and 3 (latency-bound; a K sweep: K = 1 fastest)
    assert api.grid_plan(_abi.nurbs_shape(1, 8, 8, 3, 3, 64, 64, 0))["K"] == 1
    assert api.grid_plan(_abi.nurbs_shape(1, 32, 32, 3, 3, 512, 512, 0))["K"] == 1


def test_binding_rejects_wrong_dtypes_and_sizes():
    """The Python binding checks dtype and element counts before any pointer reaches the C
    ABI (a wrong size would read out of bounds, a float64 tensor would be reinterpreted)."""
    import torch
    from paper_2104_14547_b200 import _abi, api
    sh = _abi.nurbs_shape(2, 8, 7, 3, 2, 5, 6, 0)
    good = dict(ctrl=torch.zeros(2, 8, 7, 4), U=torch.zeros(12), V=torch.zeros(10), u=torch.zeros(5),
                v=torch.zeros(6), pts_out=torch.zeros(2, 5, 6, 3), ctrl_grad=torch.zeros(2, 8, 7, 4))
    api._expect(sh, True, **good)
    api._expect(sh, ctrl_grad=torch.zeros(3, 8, 7, 4))       # a larger buffer passes the C-ABI mirrors
    with pytest.raises(ValueError):
        api._expect(sh, True, ctrl_grad=torch.zeros(3, 8, 7, 4))  # ... but not the convenience wrappers
    for key, bad in [("ctrl", torch.zeros(2, 8, 7, 4, dtype=torch.float64)), ("U", torch.zeros(11)),
                     ("V", torch.zeros(11)), ("u", torch.zeros(6)), ("pts_out", torch.zeros(2, 5, 6, 4)),
                     ("ctrl_grad", torch.zeros(1, 8, 7, 4))]:
        with pytest.raises(ValueError):
            api._expect(sh, True, **{**good, key: bad})
    kb = _abi.nurbs_shape(2, 8, 7, 3, 2, 5, 6, 1)  # batched knots: [B][n+p+1]
    api._expect(kb, True, U=torch.zeros(2, 12), V=torch.zeros(2, 10))
    with pytest.raises(ValueError):
        api._expect(kb, U=torch.zeros(12))
    with pytest.raises(ValueError):   # uv of paired points
        api._expect_points(_abi.nurbs_shape(2, 8, 7, 3, 2, 9, 1, 0), torch.zeros(2, 8, 2))
    with pytest.raises(ValueError):   # float64 is never reinterpreted
        api._expect(sh, ctrl=torch.zeros(4, 8, 7, 4, dtype=torch.float64))
    # tables built for one shape are refused for another
    t = api.Tables(_abi.nurbs_shape(4, 8, 7, 3, 2, 5, 6, 0), torch.zeros(16, dtype=torch.uint8))
    api._expect_tables(_abi.nurbs_shape(9, 8, 7, 3, 2, 5, 6, 0), t)        # another batch size is fine
    with pytest.raises(ValueError):
        api._expect_tables(_abi.nurbs_shape(4, 8, 7, 3, 2, 5, 7, 0), t)    # another n_v is not
    with pytest.raises(ValueError):
        api._expect_tables(_abi.nurbs_shape(4, 9, 7, 3, 2, 5, 6, 0), t)
