"""In-tree build of libnurbs_b200.so for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2104_14547_b200.build [--force] [-v]

The grid kernel is instantiated for every (p, q, fwd/bwd, TMA/direct) combination; its
translation unit is compiled once per row degree p (-DNB_P=p) in parallel.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnurbs_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17"] + ARCH + ["-Xcompiler", "-fPIC", "-diag-suppress", "128"]


def units():
    u = [("nurbs_api", os.path.join(CSRC, "nurbs_api.cu"), []),
         ("nurbs_kernels", os.path.join(CSRC, "nurbs_kernels.cu"), []),
         ("nurbs_derivs", os.path.join(CSRC, "nurbs_derivs.cu"), []),
         ("nurbs_points", os.path.join(CSRC, "nurbs_points.cu"), []),
         ("nurbs_knots", os.path.join(CSRC, "nurbs_knots.cu"), []),
         ("nurbs_bwd_tc", os.path.join(CSRC, "nurbs_bwd_tc.cu"), [])]
    for p in range(6):
        u.append((f"nurbs_grid_p{p}", os.path.join(CSRC, "nurbs_grid_p.cu"), [f"-DNB_P={p}"]))
    for p in range(1, 6):
        u.append((f"nurbs_points_p{p}", os.path.join(CSRC, "nurbs_points_p.cu"), [f"-DNB_P={p}"]))
    return u


def deps():
    return glob.glob(os.path.join(CSRC, "*")) + [os.path.join(ROOT, "include", "nurbs.h")]


OBJ_CACHE = os.path.join(HERE, "build_obj")  # per-unit objects keyed by a hash of their inputs


def _unit_key(src: str, flags) -> str:
    """Hash of a unit's source, every header under csrc/ + include/nurbs.h, and its flags."""
    import hashlib
    h = hashlib.sha256()
    for path in [src] + sorted(p for p in deps() if not p.endswith(".cu")):
        with open(path, "rb") as f:
            h.update(os.path.relpath(path, ROOT).encode() + b"\0" + f.read())
    h.update(" ".join(flags).encode())
    return h.hexdigest()[:24]


def build(force: bool = False, verbose: bool = False, lib: str = LIB, defines=()) -> str:
    """Compile every unit for sm_100a (units whose inputs are unchanged come from the object
    cache) and link libnurbs_b200.so. Rebuilds only when a source is newer than the library."""
    LIB_ = lib
    stale = force or not os.path.exists(LIB_) or any(os.path.getmtime(d) > os.path.getmtime(LIB_) for d in deps())
    if not stale:
        return LIB_
    os.makedirs(OBJ_CACHE, exist_ok=True)
    procs, objs = [], []
    for name, src, extra in units():
        flags = FLAGS + list(defines) + extra
        obj = os.path.join(OBJ_CACHE, f"{name}-{_unit_key(src, flags)}.o")
        objs.append(obj)
        if os.path.exists(obj) and not force:
            continue
        cmd = [NVCC] + flags + (["-Xptxas", "-v"] if verbose else []) + ["-c", src, "-o", obj + ".tmp"]
        procs.append((name, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = False
    for name, obj, pr in procs:
        out, _ = pr.communicate()
        if pr.returncode != 0:
            failed = True
            sys.stderr.write(f"--- {name}\n{out}")
        else:
            os.replace(obj + ".tmp", obj)
            if verbose:
                sys.stderr.write(out)
    if failed:
        raise RuntimeError("nvcc failed building libnurbs_b200.so")
    res = subprocess.run([NVCC] + ARCH + ["-shared", "-o", LIB_ + ".tmp"] + objs, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(LIB_ + ".tmp", LIB_)
    # keep the cache small: drop objects of units that are no longer current
    keep = {os.path.basename(o) for o in objs}
    for f in os.listdir(OBJ_CACHE):
        if f.endswith(".o") and f not in keep and not defines:
            try:
                os.remove(os.path.join(OBJ_CACHE, f))
            except OSError:
                pass
    return LIB_


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
