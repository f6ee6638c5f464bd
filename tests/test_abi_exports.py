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


def test_plan_is_bounded():
    """Row-block bands never exceed the kRMax = 16 smem rows; plans cover every span."""
    import math
    for (B, n, p, n_u, m, n_v) in [(4096, 16, 3, 128, 16, 128), (1, 256, 3, 8192, 256, 8192), (1, 8, 3, 64, 8, 64),
                                   (1, 32, 3, 512, 32, 512), (7, 40, 5, 9, 11, 300), (1, 6, 3, 100, 6, 100)]:
        spans = n - p
        K = spans if spans + p <= 16 else 16 - p
        while K > 1 and B * math.ceil(spans / K) * math.ceil(n_v / 128) < 592:
            K = (K + 1) // 2
        assert K + p <= 16 or n <= 16
        assert math.ceil(spans / K) * K >= spans
