#!/usr/bin/env python
"""Benchmark of the NURBS-Diff hot path on B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1|2|3|4|5] [--impl reference]
                    [--shard-of G] [--weak] [--ordered-reduce] [--derivs | --knots | --paired]

A step is one pass of the whole hot path over one batch: nurbs_surface_fwd (FindSpan, basis,
homogeneous banded sum, rational divide) then nurbs_surface_bwd (dL/dP, dL/dw, zero knot
gradients), through the C ABI.

* --config 4 (default; BASELINE.json configs[3]): 4096 bicubic 16x16 NURBS surfaces, 128x128
  grid each. With N GPUs the ONE batch of 4096 surfaces is sharded (rank r owns surfaces
  shard_range(4096, N, r): 512 per rank at N = 8; strong scaling, no collective). --weak
  gives every rank its own 4096 surfaces instead.
* --config 5: one 256x256 surface on the 8192^2 grid, u-rows sharded over the ranks, one NCCL
  all-reduce of the gradients (order pinned, NCCL_ALGO=Ring NCCL_PROTO=Simple), or with
  --ordered-reduce an all-gather + rank-order sum in the library (bitwise repeatable).
* --config 1 / 2: latency lines (the curve of configs[0], the 8x8 surface of configs[1]):
  microseconds per fwd and per bwd call under CUDA-graph replay.
* --config 3: the SGD surface fit of configs[2]; a step is the whole 1000-iteration fit
  (--iters), each iteration one fused step, the loop one CUDA graph.
* --shard-of G: on ONE GPU, run rank 0's shard of a G-way split (the per-rank compute of the
  N = G run, measurable without G GPUs).

`--gpus N` without torchrun re-launches this script under torch.distributed.run with N ranks
(127.0.0.1). Prints ONE JSON line on rank 0 (fields: DESIGN.md §6).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NURBS surface points/sec fwd and fwd+bwd (fp32); achieved HBM GB/s vs peak"
NOMINAL_HBM_GBS = 8000.0   # B200 HBM3e nominal (SURVEY §8(d) reports against both)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default 200; config 3: 3 fits)")
    ap.add_argument("--warmup", type=int, default=None, help="untimed steps (default 10; config 3: 3)")
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shard-of", type=int, default=0, help="one GPU: time rank 0's shard of a G-way split")
    ap.add_argument("--weak", action="store_true", help="config 4: every rank its own 4096 surfaces")
    ap.add_argument("--ordered-reduce", action="store_true", help="config 5: all-gather + rank-order sum")
    ap.add_argument("--tc", action="store_true",
                    help="time the tcgen05 (3xTF32) backward instead of the SIMT backward where it applies")
    ap.add_argument("--iters", type=int, default=1000, help="config 3: SGD iterations per fit (one step)")
    ap.add_argument("--cpu-seconds", type=float, default=8.0, help="oracle cpu_baseline budget per leg")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-chunk", type=int, default=256, help="surfaces per chunk of the pipelined e2e (config 4)")
    ap.add_argument("--derivs", action="store_true", help="time the NEXT-3 derivative kernel instead")
    ap.add_argument("--knots", action="store_true",
                    help="time the NEXT-4 backward with true knot gradients (nurbs_surface_bwd_knots) on the config")
    ap.add_argument("--paired", action="store_true",
                    help="time the NEXT-1 paired-points path on cfg4p (cfg4's nets, 16384 scattered points each)")
    a = ap.parse_args(argv)
    if a.steps is None:
        a.steps = 3 if a.config == 3 else 200
    if a.warmup is None:
        a.warmup = 3 if a.config == 3 else 10
    return a


# --------------------------------------------------------------------------- launching
def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def torchrun_cmd(n: int, argv, port: int | None = None) -> list:
    """The driver's own launch line for N ranks on one node (rendezvous on 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", "--master-port", str(port or free_port()),
            os.path.abspath(__file__)] + list(argv)


def world_info():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def host_info() -> dict:
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(kernel: str, config: int):
    """dram__bytes_read+write per launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d[f"cfg{config}"][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML samples of SM clock + clock-event reasons during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.ok = False
        self.samples, self.reasons = [], set()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- workloads
def workload_name(config):
    return {
        1: "cfg1: one cubic NURBS curve, 6 control points, clamped knots, 100 samples, fwd+bwd (configs[0])",
        2: "cfg2: one bicubic NURBS surface, 8x8 control net, random weights, 64x64 grid, fwd+bwd (configs[1])",
        3: ("cfg3: SGD surface fit, 1 bicubic NURBS 32x32 control net, 512x512 target grid, 1000 iterations, "
            "one fused fwd+MSE+bwd+update step per iteration, iterations in one CUDA graph (configs[2])"),
        4: "cfg4: 4096 bicubic NURBS surfaces x 16x16 control nets, 128x128 grid each, fwd+bwd (BASELINE.json configs[3])",
        5: "cfg5: one bicubic 256x256 NURBS surface, 8192x8192 grid, u-rows sharded, fwd+bwd+allreduce (configs[4])",
    }[config]


def grid_config(args, world: int) -> dict:
    """The `config` object of a config-4/5 line: identical for our arm and the reference arm."""
    G = world if world > 1 else max(1, args.shard_of or 1)
    if args.config == 4:
        par = (f"weak: {world} ranks x 4096 surfaces, no collective" if args.weak
               else f"batch-sharded: 4096 surfaces / {G} ranks, no collective")
        cfg = {"workload": workload_name(4), "global_batch": 4096 * (world if args.weak else 1),
               "points_per_step": 4096 * 128 * 128 * (world if args.weak else 1), "parallelism": par,
               "p": 3, "q": 3, "n": 16, "m": 16, "grid": [128, 128]}
    else:
        par = (f"u-rows sharded x{G} + " + ("all-gather + rank-order sum (nurbs_sum_partials)" if args.ordered_reduce
                                            else "NCCL all-reduce (NCCL_ALGO=Ring, NCCL_PROTO=Simple)"))
        cfg = {"workload": workload_name(5), "global_batch": 1, "points_per_step": 8192 * 8192, "parallelism": par,
               "p": 3, "q": 3, "n": 256, "m": 256, "grid": [8192, 8192]}
    if args.shard_of and world == 1:
        cfg["shard"] = f"rank 0 of a {args.shard_of}-way split, timed alone on one GPU (the per-rank compute at N = {args.shard_of})"
    cfg["tables"] = "precomputed span/basis tables (P:171)"
    cfg["l2"] = "inputs larger than L2 (out and dL/dS are 805 MB each at N = 1), no flush"
    return cfg


def local_slice(args, rank: int, world: int):
    """(first, last) unit of this rank: surfaces of config 4, u-rows of config 5."""
    from paper_2104_14547_b200 import dist as nbd
    G, r = (world, rank) if world > 1 else (max(1, args.shard_of or 1), 0)
    total = 4096 if args.config == 4 else 8192
    if args.config == 4 and args.weak:
        return 0, total
    return nbd.shard_range(total, G, r)


# --------------------------------------------------------------------------- oracle legs
def oracle_grid_leg(config: int, seconds: float, threads: int):
    """The fp64 CPU oracle (oracle/, as it stands) on distinct units of the config's workload
    (cfg4: chunks of 16 surfaces; cfg5: blocks of 64 u-rows), fwd + bwd, in unit order, until
    `seconds` of wall time are used; `threads` > 1 runs units concurrently (oracle.pmap:
    ctypes releases the GIL). Returns (points/s, description, threads, seconds)."""
    import numpy as np

    import oracle
    import workloads as wl
    oracle.build()
    if config == 4:
        w = wl.config4()
        per = 16
        n_units = w.B // per

        def unit(k):
            c = w.ctrl[k * per:(k + 1) * per]
            g = np.random.default_rng(500 + k).standard_normal((per, 128, 128, 3), dtype=np.float32)
            oracle.surface_fwd(c, w.U, w.V, w.u, w.v, w.p, w.q)
            oracle.surface_bwd(c, w.U, w.V, w.u, w.v, g, w.p, w.q)
            return per * 128 * 128
        what = "surfaces"
    else:
        w = wl.config5()
        per = 64
        n_units = w.n_u // per

        def unit(k):
            u = w.u[k * per:(k + 1) * per]
            g = np.random.default_rng(500 + k).standard_normal((1, per, 8192, 3), dtype=np.float32)
            oracle.surface_fwd(w.ctrl, w.U, w.V, u, w.v, w.p, w.q)
            oracle.surface_bwd(w.ctrl, w.U, w.V, u, w.v, g, w.p, w.q)
            return per * 8192
        what = "u-rows"
    t0 = time.perf_counter()
    done, pts = 0, 0
    while done < n_units and time.perf_counter() - t0 < seconds:
        batch = list(range(done, min(n_units, done + threads)))
        pts += sum(oracle.pmap(unit, [(k,) for k in batch], threads))
        done += len(batch)
    dt = time.perf_counter() - t0
    desc = (f"cfg{config} fwd+bwd (Form E) on {what} [0,{done * per}) of {n_units * per} "
            f"({pts} points, each unit distinct), fp64, {threads} thread(s)")
    return pts / dt, desc, threads, dt


def cpu_baseline_grid(args) -> dict:
    """Two timings: one thread, and all host cores."""
    all_c = __import__("oracle").cores()
    r1, d1, _, s1 = oracle_grid_leg(args.config, args.cpu_seconds, 1)
    rN, dN, cN, sN = oracle_grid_leg(args.config, args.cpu_seconds, all_c)
    return {"value": rN, "unit": "points/s", "cores": cN, "kind": "oracle", "sample": dN, "seconds": sN,
            "single_thread": {"value": r1, "cores": 1, "sample": d1, "seconds": s1}, **host_info()}


def run_reference(args, rank, world):
    """The reference arm of this tier: the fp64 oracle as it stands, on the host cores, on a
    bounded sample of our arm's workload per step (rank 0 only; other ranks exit 0)."""
    if rank != 0:
        return
    import numpy as np

    import oracle
    import workloads as wl
    oracle.build()
    threads = oracle.cores()
    if args.config in (4, 5):
        cfg = grid_config(args, world)
        if args.config == 4:
            w = wl.config4(B=8 * threads)
            g = np.random.default_rng(7).standard_normal((w.B, 128, 128, 3), dtype=np.float32)
            items = [(k * 8, (k + 1) * 8) for k in range(threads)]
            unit = lambda b0, b1: (oracle.surface_fwd(w.ctrl[b0:b1], w.U, w.V, w.u, w.v, 3, 3),  # noqa: E731
                                   oracle.surface_bwd(w.ctrl[b0:b1], w.U, w.V, w.u, w.v, g[b0:b1], 3, 3))
            pts = w.B * 128 * 128
            sample = f"cfg4: {w.B} of 4096 surfaces per step ({pts} points), fp64 oracle, {threads} threads"
        else:
            w = wl.config5()
            rows = 8
            g = np.random.default_rng(7).standard_normal((1, rows * threads, 8192, 3), dtype=np.float32)
            items = [(k * rows, (k + 1) * rows) for k in range(threads)]
            unit = lambda a0, a1: (oracle.surface_fwd(w.ctrl, w.U, w.V, w.u[a0:a1], w.v, 3, 3),  # noqa: E731
                                   oracle.surface_bwd(w.ctrl, w.U, w.V, w.u[a0:a1], w.v, g[:, a0:a1], 3, 3))
            pts = rows * threads * 8192
            sample = f"cfg5: {rows * threads} of 8192 u-rows per step ({pts} points), fp64 oracle, {threads} threads"
        step = lambda: oracle.pmap(unit, items, threads)  # noqa: E731
        metric, unit_name = METRIC, "points/s"
    else:
        cfg = {"workload": workload_name(args.config)}
        step, pts, sample = _oracle_small_step(args.config, args.iters)
        metric, unit_name, threads = METRIC, "points/s", 1
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = pts * args.steps / dt
    line = {"metric": metric, "value": value, "unit": unit_name, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak" if (args.config == 4 and args.weak) else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": unit_name, "cores": threads, "kind": "oracle", "sample": sample,
                             **host_info()},
            "e2e": {"value": value, "unit": unit_name, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _oracle_small_step(config: int, iters: int):
    """Oracle step for configs 1-3 (one small problem, one thread). Config 3: a bounded number
    of fit iterations per step (the full 1000 would take minutes)."""
    import numpy as np

    import oracle
    import workloads as wl
    oracle.build()
    if config == 1:
        c = wl.config1()
        g = c.grad_out()
        return (lambda: (oracle.curve_fwd(c.ctrl, c.U, c.u, c.p), oracle.curve_bwd(c.ctrl, c.U, c.u, g, c.p))), 100, \
            "cfg1 fwd+bwd, fp64 oracle, 1 thread"
    if config == 2:
        w = wl.config2()
        g = w.grad_out(0)
        return (lambda: (oracle.surface_fwd(w.ctrl, w.U, w.V, w.u, w.v, 3, 3),
                         oracle.surface_bwd(w.ctrl, w.U, w.V, w.u, w.v, g, 3, 3))), 4096, \
            "cfg2 fwd+bwd, fp64 oracle, 1 thread"
    truth, init = wl.config3_fit()
    T = oracle.surface_fwd(truth.ctrl, truth.U, truth.V, truth.u, truth.v, 3, 3)
    state = {"c": init.ctrl.astype(np.float64)}
    k = 5

    def step():
        for _ in range(k):
            S = oracle.surface_fwd(state["c"], truth.U, truth.V, truth.u, truth.v, 3, 3)
            d = S - T
            gr = oracle.surface_bwd(state["c"], truth.U, truth.V, truth.u, truth.v, 2 * d / d[..., 0].size, 3, 3)
            state["c"] = state["c"] - 200.0 * gr
    return step, k * 512 * 512, f"cfg3: {k} fit iterations (fwd+MSE+bwd+SGD) per step at 512x512, fp64 oracle, 1 thread"


# --------------------------------------------------------------------------- config 1 / 2: latency
def run_latency(args, rank, world):
    """Configs 1 and 2: latency-bound single problems. Reported: microseconds
    per fwd call and per bwd call inside a CUDA graph of `G` back-to-back calls (graph launch
    amortised), the fwd+bwd step rate, and e2e through the public API with host buffers."""
    import numpy as np
    import torch

    import paper_2104_14547_b200 as nb
    import workloads as wl
    local = world_info()[2]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    T_ = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    if args.config == 1:
        c = wl.config1()
        ctrl, U, u, gout = T_(c.ctrl), T_(c.U), T_(c.u), T_(c.grad_out())
        sh = nb.curve_shape(ctrl, U, u, c.p)
        out = torch.empty((1, 100, 3), device=dev)
        grad = torch.empty_like(ctrl)
        gU = torch.empty_like(U)
        tab = nb.Tables.build(sh, U, None, u, None)
        fwd = lambda s: nb.nurbs_curve_fwd(sh, ctrl, U, u, tab, out, s)  # noqa: E731
        bwd = lambda s: nb.nurbs_curve_bwd(sh, ctrl, U, u, tab, gout, grad, gU, None, 0, s)  # noqa: E731
        pts, host_in = 100, (c.ctrl, c.grad_out())
    else:
        w = wl.config2()
        ctrl, U, V, u, v, gout = T_(w.ctrl), T_(w.U), T_(w.V), T_(w.u), T_(w.v), T_(w.grad_out(0))
        sh = nb.surface_shape(ctrl, U, u, v, 3, 3)
        out = torch.empty((1, 64, 64, 3), device=dev)
        grad = torch.empty_like(ctrl)
        gU, gV = torch.empty_like(U), torch.empty_like(V)
        tab = nb.Tables.build(sh, U, V, u, v)
        wsb = nb.bwd_workspace_bytes(sh)   # the plan tiles this small net (cross-tile reduce)
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        fwd = lambda s: nb.nurbs_surface_fwd(sh, ctrl, U, V, u, v, tab, out, s)  # noqa: E731
        bwd = lambda s: nb.nurbs_surface_bwd(sh, ctrl, U, V, u, v, tab, gout, grad, gU, gV, ws, wsb, s)  # noqa: E731
        pts, host_in = 4096, (w.ctrl, w.grad_out(0))
    G = 100
    s = torch.cuda.Stream(dev)

    def graph_of(fn):
        s.wait_stream(torch.cuda.current_stream())
        fn(s)                      # warm (first-launch attribute setup) outside the capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(G):
                fn(s)
        return g

    g_f, g_b = graph_of(fwd), graph_of(bwd)
    g_fb = graph_of(lambda st: (fwd(st), bwd(st)))

    def time_graph(g):
        for _ in range(args.warmup):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / (args.steps * G) * 1e3   # us per call (or per pair)

    sampler = ClockSampler(local)
    with sampler:
        us_f, us_b, us_fb = time_graph(g_f), time_graph(g_b), time_graph(g_fb)
    # e2e: pinned host ctrl + dL/dS -> device, fwd + bwd through the public calls, S + grad -> host
    h_ctrl = torch.from_numpy(host_in[0].copy()).pin_memory()
    h_g = torch.from_numpy(host_in[1].copy()).pin_memory()
    h_out = torch.empty(out.shape).pin_memory()
    h_grad = torch.empty(grad.shape).pin_memory()
    cur = torch.cuda.current_stream()

    def e2e_step():
        ctrl.copy_(h_ctrl, non_blocking=True)
        gout.copy_(h_g, non_blocking=True)
        fwd(cur)
        bwd(cur)
        h_out.copy_(out, non_blocking=True)
        h_grad.copy_(grad, non_blocking=True)

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    E = max(args.steps, 50)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(E):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    e2e_us = e0.elapsed_time(e1) / E * 1e3
    cpu = None
    if not args.no_cpu_baseline:
        step, cpts, sample = _oracle_small_step(args.config, args.iters)
        t0, k = time.perf_counter(), 0
        while time.perf_counter() - t0 < min(args.cpu_seconds, 3.0) or k < 3:
            step()
            k += 1
        dt = time.perf_counter() - t0
        cpu = {"value": cpts * k / dt, "unit": "points/s", "cores": 1, "kind": "oracle",
               "sample": f"{sample}, {k} steps", "us_per_fwd_bwd": dt / k * 1e6, **host_info()}
    if rank == 0:
        line = {"metric": METRIC, "value": pts / (us_fb * 1e-6), "unit": "points/s", "n_gpus": 1,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": us_fb * 1e-3, "higher_is_better": True,
                "scaling": "replicas only", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": workload_name(args.config), "points_per_step": pts,
                           "timing": f"CUDA graph of {G} calls replayed {args.steps} times; per-call time"},
                "fwd_us": us_f, "bwd_us": us_b, "fwd_bwd_us": us_fb,
                "roofline": {"bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None,
                             "traffic": None, "note": f"{pts} points per call: launch/latency bound, no % of HBM"},
                "cpu_baseline": cpu,
                "e2e": {"value": pts / (e2e_us * 1e-6), "unit": "points/s", "us_per_step": e2e_us,
                        "h2d_bytes_per_step": host_in[0].nbytes + host_in[1].nbytes,
                        "d2h_bytes_per_step": out.numel() * 4 + grad.numel() * 4},
                "gpu_launches": 2 * G * args.steps * 3, "clocks": sampler.summary()}
        print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- config 3: fitting loop
def run_fit(args, rank, world):
    """Config 3: a step is the whole --iters (1000) SGD iteration fit of the
    fused fitting step, recorded in one CUDA graph and replayed; inputs resident in HBM (the
    3 MB target stays L2-resident across iterations: the loop is latency-bound)."""
    import numpy as np
    import torch

    import paper_2104_14547_b200 as nb
    import workloads as wl
    local = world_info()[2]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    truth, init = wl.config3_fit()
    T_ = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    U, V, u, v = T_(truth.U), T_(truth.V), T_(truth.u), T_(truth.v)
    sh = nb.nurbs_shape(1, 32, 32, 3, 3, 512, 512, 0)
    tables = nb.Tables.build(sh, U, V, u, v)
    target = nb.surface_fwd(T_(truth.ctrl), U, V, u, v, 3, 3, tables=tables)  # synthetic target
    ctrl = T_(init.ctrl)
    fitter = nb.SurfaceFitter(ctrl, U, V, u, v, target, 3, 3, lr=200.0, tables=tables)
    I = args.iters
    fitter.run(I)            # records the graph and runs it once
    for _ in range(max(0, args.warmup - 1)):
        ctrl.copy_(T_(init.ctrl))
        fitter.run(I)
    torch.cuda.synchronize()
    K = args.steps
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * K)]
    sampler = ClockSampler(local)
    init_d = T_(init.ctrl)
    with sampler:
        for k in range(K):
            ctrl.copy_(init_d)          # every step is the same fit from the same start
            ev[2 * k].record()
            losses = fitter.run(I)
            ev[2 * k + 1].record()
        torch.cuda.synchronize()
    ms_fit = sum(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(K)) / K
    lh = losses.cpu().numpy()
    pts = 512 * 512
    # e2e: host ctrl + target -> device, the 1000-iteration fit, fitted ctrl + losses -> host
    h_c = torch.from_numpy(init.ctrl.copy()).pin_memory()
    h_target = target.cpu().pin_memory()
    h_out = torch.empty(ctrl.shape, dtype=torch.float32).pin_memory()
    h_loss = torch.empty(I, dtype=torch.float32).pin_memory()
    d_t = torch.empty_like(target)
    E = 3
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(E):
        ctrl.copy_(h_c, non_blocking=True)
        d_t.copy_(h_target, non_blocking=True)
        target.copy_(d_t)       # the fitter reads `target`; same bytes, refreshed each step
        fitter.run(I)
        h_out.copy_(ctrl, non_blocking=True)
        h_loss.copy_(fitter.losses, non_blocking=True)
    e3.record()
    torch.cuda.synchronize()
    e2e_ms = e2.elapsed_time(e3) / E
    cpu = None
    if not args.no_cpu_baseline:
        step, cpts, sample = _oracle_small_step(3, I)
        t0, k = time.perf_counter(), 0
        while time.perf_counter() - t0 < args.cpu_seconds or k < 1:
            step()
            k += 1
        dt = time.perf_counter() - t0
        cpu = {"value": cpts * k / dt, "unit": "points/s", "cores": 1, "kind": "oracle",
               "sample": f"{sample}, {k} steps", "it_per_s": cpts * k / pts / dt, **host_info()}
    line = {
        "metric": METRIC, "value": pts * I / (ms_fit * 1e-3), "unit": "points/s", "n_gpus": 1, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_fit, "higher_is_better": True, "scaling": "replicas only",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded ground-truth NURBS target; init P*+N(0,0.05), w=1)",
        "config": {"workload": workload_name(3), "lr": 200.0, "iterations_per_step": I,
                   "l2": "target (3 MB) L2-resident across iterations by design of the loop"},
        "it_per_s": I / (ms_fit * 1e-3), "us_per_iteration": ms_fit * 1e3 / I,
        "seconds_per_1000_iterations": ms_fit * 1e-3 * 1000 / I,
        "loss_first_last": [float(lh[0]), float(lh[-1])],
        "paper_context": "Ducky fit, 14x13 net at 512^2: 1000 iterations in < 2 minutes (>= 8.3 it/s), hardware unstated (P:480)",
        "roofline": {"bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None, "traffic": None,
                     "note": "2 launches per iteration (fused step + update) on a 262K-point problem"},
        "cpu_baseline": cpu,
        "e2e": {"value": pts * I / (e2e_ms * 1e-3), "unit": "points/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": init.ctrl.nbytes + target.numel() * 4,
                "d2h_bytes_per_step": init.ctrl.nbytes + I * 4},
        "gpu_launches": 2 * I * K,
        "clocks": sampler.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- NEXT-3 derivatives
def run_derivs(args, rank, world):
    """NEXT-3: S, S_u, S_v and unit normals on config 4's workload (48 B/point written)."""
    import numpy as np
    import torch

    import paper_2104_14547_b200 as nb
    import workloads as wl
    local = world_info()[2]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w = wl.config4() if args.config == 4 else wl.config5()
    T_ = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    ctrl, U, V, u, v = T_(w.ctrl), T_(w.U), T_(w.V), T_(w.u), T_(w.v)
    sh = nb.nurbs_shape(w.B, w.n, w.m, w.p, w.q, w.n_u, w.n_v, 0)
    outs = [torch.empty((w.B, w.n_u, w.n_v, 3), dtype=torch.float32, device=dev) for _ in range(4)]
    run = lambda: nb.nurbs_surface_derivs(sh, ctrl, U, V, u, v, outs[0], outs[1], outs[2], outs[3])  # noqa: E731
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        e0.record()
        for _ in range(args.steps):
            run()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    pts = w.points
    byts = pts * 48 + w.ctrl.nbytes
    peak, kind = load_peaks()
    line = {"metric": "NURBS surface points/sec with parametric derivatives and normals (fp32, NEXT-3)",
            "value": pts / (ms * 1e-3), "unit": "points/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": workload_name(args.config) + " -> S, S_u, S_v, normals"},
            "roofline": {"bound": "hbm", "achieved": byts / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": byts / (ms * 1e-3) / 1e9 / peak, "frac_nominal": byts / (ms * 1e-3) / 1e9 / NOMINAL_HBM_GBS,
                         "traffic": None, "algorithmic_bytes_per_launch": byts, "peak_kind": kind},
            "gpu_launches": args.steps, "clocks": sampler.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- NEXT-4 knot gradients
def run_knots(args, rank, world):
    """NEXT-4: nurbs_surface_bwd_knots (control AND true knot gradients) on config 4 / 5,
    timed beside the plain backward (the knot gradients' extra cost)."""
    import numpy as np
    import torch

    import paper_2104_14547_b200 as nb
    import workloads as wl
    local = world_info()[2]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w = wl.config4() if args.config == 4 else wl.config5()
    T_ = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    ctrl, U, V, u, v = T_(w.ctrl), T_(w.U), T_(w.V), T_(w.u), T_(w.v)
    sh = nb.nurbs_shape(w.B, w.n, w.m, w.p, w.q, w.n_u, w.n_v, 0)
    tables = nb.Tables.build(sh, U, V, u, v)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    gout = torch.randn((w.B, w.n_u, w.n_v, 3), dtype=torch.float32, device=dev, generator=gen)
    grad = torch.empty_like(ctrl)
    gU, gV = torch.empty_like(U), torch.empty_like(V)
    wsk = nb.knots_workspace_bytes(sh)
    work = torch.empty(wsk, dtype=torch.uint8, device=dev)
    wsb = nb.bwd_workspace_bytes(sh)
    workb = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    kg = lambda: nb.nurbs_surface_bwd_knots(sh, ctrl, U, V, u, v, tables, gout, grad, gU, gV, work, wsk)  # noqa: E731
    plain = lambda: nb.nurbs_surface_bwd(sh, ctrl, U, V, u, v, tables, gout, grad, gU, gV, workb, wsb)  # noqa: E731

    def timeit(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.steps

    sampler = ClockSampler(local)
    with sampler:
        ms = timeit(kg)
        ms_plain = timeit(plain)
    pts = w.points
    byts = pts * 12 + 2 * w.ctrl.nbytes
    peak, kind = load_peaks()
    line = {"metric": "NURBS surface points/sec of the backward with true knot gradients (fp32, NEXT-4)",
            "value": pts / (ms * 1e-3), "unit": "points/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": workload_name(args.config) + " -> dL/dP, dL/dw, dL/dU, dL/dV"},
            "plain_bwd_ms": ms_plain, "cost_vs_plain_bwd": ms / ms_plain,
            "roofline": {"bound": "hbm", "achieved": byts / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": byts / (ms * 1e-3) / 1e9 / peak, "traffic": None,
                         "algorithmic_bytes_per_launch": byts, "peak_kind": kind},
            "gpu_launches": args.steps * (7 if wsb == 0 else 8), "clocks": sampler.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- NEXT-1 paired points
FP32_FMA_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4: FFMA2 fma-pipe peak at clocks.max.sm


def paired_flops_per_point(p, q, bwd):
    """Algorithmic flops of one paired point: A2.2 basis per direction
    sum_j (2 + 4j), the separable homogeneous sum 8((p+1)(q+1) + (p+1)), divide 4; the
    backward adds G (10) and the (p+1)(q+1) float4 accumulations 8(p+1)(q+1) + 4(p+1)."""
    basis = sum(2 + 4 * j for j in range(1, p + 1)) + sum(2 + 4 * j for j in range(1, q + 1))
    fwd = basis + 8 * ((p + 1) * (q + 1) + (p + 1)) + 4
    return fwd + (10 + 8 * (p + 1) * (q + 1) + 4 * (p + 1) if bwd else 0)


def run_paired(args, rank, world):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2104_14547_b200 as nb
    from paper_2104_14547_b200 import dist as nbd
    import workloads as wl
    local = world_info()[2]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        nbd.init_nccl(dev)
    full = wl.config4_paired(seed=41)
    b0, b1 = nbd.shard_range(full.B, world, rank) if world > 1 else (0, full.B)
    T_ = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    ctrl, U, V, uv = T_(full.ctrl[b0:b1]), T_(full.U), T_(full.V), T_(full.uv[b0:b1])
    g_host = full.grad_out()[b0:b1]
    gout = T_(g_host)
    B = b1 - b0
    sh = nb.nurbs_shape(B, full.n, full.m, full.p, full.q, full.N, 1, 0)
    out = torch.empty((B, full.N, 3), dtype=torch.float32, device=dev)
    grad = torch.empty_like(ctrl)
    gU, gV = torch.empty_like(U), torch.empty_like(V)
    ws_bytes = nb.points_workspace_bytes(sh)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    fwd = lambda: nb.nurbs_surface_points_fwd(sh, ctrl, U, V, uv, out, stream)  # noqa: E731
    bwd = lambda: nb.nurbs_surface_points_bwd(sh, ctrl, U, V, uv, gout, grad, gU, gV, ws, ws_bytes, stream)  # noqa: E731
    for _ in range(args.warmup):
        fwd(); bwd()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    K = args.steps
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * K + 1)]
    sampler = ClockSampler(local)
    with sampler:
        ev[0].record(stream)
        for k in range(K):
            fwd()
            ev[2 * k + 1].record(stream)
            bwd()
            ev[2 * k + 2].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([ev[0].elapsed_time(ev[2 * K]),
                      sum(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(K)) / K,
                      sum(ev[2 * k + 1].elapsed_time(ev[2 * k + 2]) for k in range(K)) / K],
                     dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, fwd_ms, bwd_ms = t.tolist()
    ms = total_ms / K
    pts = B * full.N
    all_pts = full.B * full.N
    hbm_peak, peak_kind = load_peaks()
    ctrl_b = B * full.n * full.m * 16
    fwd_bytes = pts * 20 + ctrl_b                          # uv 8 + out 12 per point
    bwd_bytes = pts * 20 + 2 * ctrl_b + ws_bytes * 2       # uv 8 + dL/dS 12; ctrl in, grad out
    fl_f, fl_b = paired_flops_per_point(full.p, full.q, False), paired_flops_per_point(full.p, full.q, True)

    def legs(ms_, byts, fl):
        gbs = byts / (ms_ * 1e-3) / 1e9
        tf = pts * fl / (ms_ * 1e-3) / 1e12
        return {"ms": ms_, "bytes": byts, "gbs": gbs, "hbm_frac": gbs / hbm_peak, "flops_per_point": fl,
                "tflops": tf, "alu_frac": tf / FP32_FMA_TFLOPS}
    lf, lb = legs(fwd_ms, fwd_bytes, fl_f), legs(bwd_ms, bwd_bytes, fl_b)
    dom, dname = (lb, "nurbs_points_bwd_kernel<3,3>") if bwd_ms >= fwd_ms else (lf, "nurbs_points_fwd_kernel<3,3>")
    if dom["alu_frac"] >= dom["hbm_frac"]:
        roof = {"bound": "alu", "achieved": dom["tflops"], "peak": FP32_FMA_TFLOPS, "unit": "TFLOP/s",
                "frac": dom["alu_frac"], "peak_kind": "fp32 FFMA2 fma-pipe: 148 SMs x 128 lanes x 2 x 1.965 GHz"}
    else:
        roof = {"bound": "hbm", "achieved": dom["gbs"], "peak": hbm_peak, "unit": "GB/s", "frac": dom["hbm_frac"],
                "peak_kind": f"{peak_kind} copy bandwidth"}
    roof.update({"kernel": dname, "traffic": None, "fwd": lf, "bwd": lb})
    # e2e: pinned host uv + dL/dS -> device, fwd + bwd, S + grad -> host (public calls)
    e2e = None
    if not args.no_e2e:
        h_uv = torch.from_numpy(np.ascontiguousarray(full.uv[b0:b1])).pin_memory()
        h_g = torch.from_numpy(np.ascontiguousarray(g_host)).pin_memory()
        h_ctrl = torch.from_numpy(np.ascontiguousarray(full.ctrl[b0:b1])).pin_memory()
        h_out = torch.empty(out.shape).pin_memory()
        h_grad = torch.empty(grad.shape).pin_memory()
        s_up, s_down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_g, ev_f, ev_o, ev_b = (torch.cuda.Event() for _ in range(4))
        first = [True]

        def e2e_step():
            if not first[0]:
                s_up.wait_event(ev_b)
                stream.wait_event(ev_o)
            first[0] = False
            with torch.cuda.stream(s_up):
                gout.copy_(h_g, non_blocking=True)
            ev_g.record(s_up)
            ctrl.copy_(h_ctrl, non_blocking=True)
            uv.copy_(h_uv, non_blocking=True)
            fwd()
            ev_f.record(stream)
            s_down.wait_event(ev_f)
            with torch.cuda.stream(s_down):
                h_out.copy_(out, non_blocking=True)
            ev_o.record(s_down)
            stream.wait_event(ev_g)
            bwd()
            ev_b.record(stream)
            h_grad.copy_(grad, non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        E = args.e2e_steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(E):
            e2e_step()
        stream.wait_event(ev_o)
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = te.item() / E
        e2e = {"value": all_pts / (e2e_ms * 1e-3), "unit": "points/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": h_uv.numel() * 4 + h_g.numel() * 4 + h_ctrl.numel() * 4,
               "d2h_bytes_per_step": h_out.numel() * 4 + h_grad.numel() * 4,
               "note": "pinned host ctrl, uv, dL/dS -> device, fwd+bwd via the C ABI, S + grad -> host; "
                       "dL/dS upload and S download overlapped with the kernels (two copy streams)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        thr = oracle.cores()

        def unit(k0, k1):
            oracle.surface_fwd_points(full.ctrl[k0:k1], full.U, full.V, full.uv[k0:k1], full.p, full.q)
            oracle.surface_bwd_points(full.ctrl[k0:k1], full.U, full.V, full.uv[k0:k1], g_host[k0:k1], full.p, full.q)
            return (k1 - k0) * full.N

        def leg(threads):
            t0, done, pts_ = time.perf_counter(), 0, 0
            while done < full.B and time.perf_counter() - t0 < args.cpu_seconds:
                items = [(done + 4 * i, done + 4 * (i + 1)) for i in range(threads) if done + 4 * (i + 1) <= full.B]
                pts_ += sum(oracle.pmap(unit, items, threads))
                done += 4 * len(items)
            return pts_ / (time.perf_counter() - t0), done, time.perf_counter() - t0
        r1, d1, s1 = leg(1)
        rN, dN, sN = leg(thr)
        cpu = {"value": rN, "unit": "points/s", "cores": thr, "kind": "oracle",
               "sample": f"cfg4p fwd+bwd on surfaces [0,{dN}) of 4096 ({dN * full.N} points), fp64, {thr} threads",
               "seconds": sN, "single_thread": {"value": r1, "cores": 1, "seconds": s1,
                                                "sample": f"surfaces [0,{d1}), 1 thread"}, **host_info()}
    if rank == 0:
        line = {"metric": "NURBS surface points/sec fwd+bwd at paired (scattered) parameter points (fp32, NEXT-1)",
                "value": all_pts / (ms * 1e-3), "unit": "points/s", "n_gpus": world, "steps": K,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (cfg4 lattice nets, uv ~ U(0,1)^2 with knot hits, N(0,1) dL/dS)",
                "config": {"workload": "cfg4p: 4096 bicubic 16x16 NURBS surfaces x 16384 scattered (u,v) points, fwd+bwd",
                           "points_per_step": all_pts, "parallelism": f"batch-sharded: 4096 / {world}, no collective",
                           "l2": "inputs larger than L2 (uv 537 MB, out and dL/dS 805 MB each), no flush"},
                "fwd_points_per_s": all_pts / (fwd_ms * 1e-3), "fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": K * (2 + (1 if ws_bytes > 0 else 0)), "clocks": sampler.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# --------------------------------------------------------------------------- configs 4 / 5: our arm
def run_grid(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_2104_14547_b200 as nb
    from paper_2104_14547_b200 import dist as nbd
    import workloads as wl

    # NB_BENCH_SHARE_GPU=1 (plumbing check only): N ranks on the visible GPUs round-robin, with a
    # gloo group (NCCL refuses two ranks on one GPU); timings are then not scaling numbers
    share = os.environ.get("NB_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            nbd.init_nccl(dev)   # async error handling + timeout; all-reduce order pinned
    assert args.warmup >= 3, "timing rules need >= 3 warm-up steps"
    if args.tc:
        nb.path_flags(tc=True).__enter__()

    hbm_peak, peak_kind = load_peaks()
    stream = torch.cuda.current_stream()

    # ---------------- this rank's share of the ONE workload (seeded, synthetic, resident in HBM)
    lo, hi = local_slice(args, rank, world)
    if args.config == 4:
        w = wl.config4(seed=4 + (1000 * rank if args.weak else 0))
        B, n, m, n_u, n_v = hi - lo, w.n, w.m, w.n_u, w.n_v
        ctrl_np, u_np = w.ctrl[lo:hi], w.u
    else:
        w = wl.config5()
        B, n, m, n_v = w.B, w.n, w.m, w.n_v
        ctrl_np, u_np = w.ctrl, w.u[lo:hi]
        n_u = hi - lo
    U_np, r0, r1 = w.U, 0, w.n
    if args.config == 5 and (hi - lo) < w.n_u:
        # point sharding: the rank evaluates its u-slab on the sub-net of the control rows its
        # knot spans touch (local support, dist.row_window): same spans, same knots, same S
        r0, r1 = nbd.row_window(w.U, w.p, w.n, float(u_np[0]), float(u_np[-1]))
        ctrl_np, U_np, n = w.ctrl[:, r0:r1], w.U[r0:r1 + w.p + 1], r1 - r0
    T = lambda a: torch.from_numpy(a.copy()).to(dev)  # noqa: E731
    ctrl, U, V, u, v = T(ctrl_np), T(U_np), T(w.V), T(u_np), T(w.v)
    sh = nb.nurbs_shape(B, n, m, w.p, w.q, n_u, n_v, 0)
    tables = nb.Tables.build(sh, U, V, u, v)
    out = torch.empty((B, n_u, n_v, 3), dtype=torch.float32, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + lo)              # a function of the unit range: same dL/dS whatever N
    gout = torch.randn((B, n_u, n_v, 3), dtype=torch.float32, device=dev, generator=gen)
    gb = nbd.GradBuffer.alloc(B, w.n, m, w.U.size, V.numel(), dev)
    windowed = (r0, r1) != (0, w.n)
    g_ctrl, g_U = gb.grad_ctrl[:, r0:r1], gb.grad_U[r0:r1 + w.p + 1]   # B = 1: contiguous views
    ws_bytes = nb.bwd_workspace_bytes(sh)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    try:
        plan = nb.grid_plan(sh)
    except AttributeError:      # an older library under NURBS_B200_LIB_EXPERIMENT (A/B timing)
        plan = None
    reducer = nbd.OrderedReducer(gb) if (world > 1 and args.config == 5 and args.ordered_reduce) else None
    launches_per_step = 2 + (1 if ws_bytes > 0 else 0) + (1 if reducer is not None else 0)
    points = B * n_u * n_v                      # this rank's points per step

    def fwd():
        nb.nurbs_surface_fwd(sh, ctrl, U, V, u, v, tables, out, stream)

    def bwd():
        if windowed:    # rows outside the window are zero in this rank's partial
            gb.flat.zero_()
        nb.nurbs_surface_bwd(sh, ctrl, U, V, u, v, tables, gout, g_ctrl, g_U, gb.grad_V, ws,
                             ws_bytes, stream)

    def reduce():
        if world > 1 and args.config == 5:
            nbd.allreduce_grads(gb, reducer=reducer)

    for _ in range(args.warmup):
        fwd(); bwd(); reduce()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---------------- timed region: K steps, events between launches on the launching stream
    K = args.steps
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * K + 1)]
    sampler = ClockSampler(local)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with sampler:
        ev[0].record(stream)
        for k in range(K):
            fwd()
            ev[3 * k + 1].record(stream)
            bwd()
            ev[3 * k + 2].record(stream)
            reduce()
            ev[3 * k + 3].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = ev[0].elapsed_time(ev[3 * K])
    fwd_ms = sum(ev[3 * k].elapsed_time(ev[3 * k + 1]) for k in range(K)) / K
    bwd_ms = sum(ev[3 * k + 1].elapsed_time(ev[3 * k + 2]) for k in range(K)) / K
    red_ms = sum(ev[3 * k + 2].elapsed_time(ev[3 * k + 3]) for k in range(K)) / K
    t = torch.tensor([total_ms, fwd_ms, bwd_ms, red_ms], dtype=torch.float64, device="cpu" if share else dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, fwd_ms, bwd_ms, red_ms = t.tolist()
    ms_per_step = total_ms / K
    # whole-job points per step: every rank's units (one rank's shard with --shard-of)
    all_points = points * world if (args.config == 4 and args.weak) else (
        (4096 * 128 * 128 if args.config == 4 else 8192 * 8192) if world > 1 else points)
    value = all_points / (ms_per_step * 1e-3)
    fwd_value = all_points / (fwd_ms * 1e-3)

    # ---------------- roofline of the dominant kernel (algorithmic bytes)
    ctrl_bytes = B * n * m * 16
    tab_bytes = (n_u + n_v) * 20
    fwd_bytes = points * 12 + ctrl_bytes + tab_bytes
    bwd_bytes = points * 12 + 2 * ctrl_bytes + tab_bytes + (U.numel() + V.numel()) * 4
    if bwd_ms >= fwd_ms:
        kname = ("nb::tc::nurbs_bwd_tc_kernel<3,3,16,IO> (bwd)" if args.tc
                 else "nurbs_grid_kernel<3,3,true,IO,false,false> (bwd)")
        kbytes, kms = bwd_bytes, bwd_ms
    else:
        kname, kbytes, kms = "nurbs_grid_kernel<3,3,false,IO,false,false> (fwd)", fwd_bytes, fwd_ms
    achieved = kbytes / (kms * 1e-3) / 1e9
    traffic = load_traffic("bwd" if "bwd" in kname else "fwd", args.config) if (world == 1 and not args.shard_of) else None
    step_bytes = fwd_bytes + bwd_bytes
    roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "frac_nominal": achieved / NOMINAL_HBM_GBS, "traffic": traffic,
                "algorithmic_bytes_per_launch": kbytes,
                "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs); frac_nominal vs 8 TB/s",
                "fwd": {"ms": fwd_ms, "bytes": fwd_bytes, "gbs": fwd_bytes / (fwd_ms * 1e-3) / 1e9,
                        "frac": fwd_bytes / (fwd_ms * 1e-3) / 1e9 / hbm_peak},
                "bwd": {"ms": bwd_ms, "bytes": bwd_bytes, "gbs": bwd_bytes / (bwd_ms * 1e-3) / 1e9,
                        "frac": bwd_bytes / (bwd_ms * 1e-3) / 1e9 / hbm_peak},
                "step": {"ms": fwd_ms + bwd_ms, "bytes": step_bytes,
                         "gbs": step_bytes / ((fwd_ms + bwd_ms) * 1e-3) / 1e9,
                         "frac": step_bytes / ((fwd_ms + bwd_ms) * 1e-3) / 1e9 / hbm_peak}}

    # ---------------- the tcgen05 backward (3xTF32, nurbs_bwd_tc.cu) timed beside the SIMT one
    tc_line = None
    if not args.tc and world == 1 and args.config == 4:
        with nb.path_flags(tc=True):
            for _ in range(3):
                bwd()
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            for _ in range(min(K, 50)):
                bwd()
            t1.record(stream)
            torch.cuda.synchronize()
        tc_ms = t0.elapsed_time(t1) / min(K, 50)
        tc_line = {"kernel": "nb::tc::nurbs_bwd_tc_kernel<3,3,16,IO> (tcgen05.mma kind::tf32, 3xTF32)", "ms": tc_ms,
                   "gbs": bwd_bytes / (tc_ms * 1e-3) / 1e9, "frac": bwd_bytes / (tc_ms * 1e-3) / 1e9 / hbm_peak,
                   "note": "opt-in path (NURBS_TC=1 / path_flags(tc=True)); the SIMT backward is the default"}

    # ---------------- e2e: host buffers through the public API, copies inside the timed region
    e2e = None
    if not args.no_e2e and args.config == 4:
        # host batch through the public pipelined API (HostBatchPipeline): chunks of surfaces,
        # uploads / kernels / downloads on three streams, both PCIe directions busy
        h_ctrl = ctrl.cpu().pin_memory()
        h_gout = gout.cpu().pin_memory()
        h_out = torch.empty(out.shape, dtype=torch.float32).pin_memory()
        h_grad = torch.empty(ctrl.shape, dtype=torch.float32).pin_memory()
        chunk = min(args.e2e_chunk, B)
        pipe = nb.HostBatchPipeline(n, m, w.p, w.q, U, V, u, v, tables, chunk=chunk, device=dev)
        for _ in range(2):
            pipe.fwd_bwd(h_ctrl, h_gout, h_out, h_grad, stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        E = args.e2e_steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(E):
            pipe.fwd_bwd(h_ctrl, h_gout, h_out, h_grad, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cpu" if share else dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = te.item() / E
        # the PCIe ceiling of this step: the same byte volumes copied both ways at once (no
        # kernels), pinned host buffers on two streams (scripts/pcie_probe.py measures it alone)
        s_a, s_b = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

        def copies():
            s_a.wait_stream(stream)
            s_b.wait_stream(stream)
            with torch.cuda.stream(s_a):
                gout.copy_(h_gout, non_blocking=True)
                ctrl.copy_(h_ctrl, non_blocking=True)
            with torch.cuda.stream(s_b):
                h_out.copy_(out, non_blocking=True)
                h_grad.copy_(ctrl, non_blocking=True)
            stream.wait_stream(s_a)
            stream.wait_stream(s_b)

        copies()
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for _ in range(3):
            copies()
        c1.record(stream)
        torch.cuda.synchronize()
        ceil_ms = c0.elapsed_time(c1) / 3
        e2e = {"value": all_points / (e2e_ms * 1e-3), "unit": "points/s", "h2d_bytes_per_step": pipe.h2d_bytes(B),
               "d2h_bytes_per_step": pipe.d2h_bytes(B), "ms_per_step": e2e_ms,
               "pcie_ceiling": {"ms_per_step": ceil_ms, "value": all_points / (ceil_ms * 1e-3),
                                "frac": ceil_ms / e2e_ms,
                                "note": "the step's h2d and d2h bytes copied both ways at once, no kernels"},
               "note": f"pinned host ctrl+grad_out -> device, fwd+bwd via the C ABI, out+grad_ctrl -> host; "
                       f"HostBatchPipeline, chunks of {chunk} surfaces on h2d/compute/d2h streams (per rank)"}
    elif not args.no_e2e:
        h_ctrl = ctrl.cpu().pin_memory()
        h_gout = gout.cpu().pin_memory()
        h_out = torch.empty(out.shape, dtype=torch.float32).pin_memory()
        h_grad = torch.empty(gb.flat.shape, dtype=torch.float32).pin_memory()
        d_ctrl = torch.empty_like(ctrl)
        d_gout = torch.empty_like(gout)
        # the forward does not need dL/dS: upload dL/dS on one copy stream while the forward
        # runs and its output downloads on another (the two PCIe directions overlap); the
        # backward waits for the upload
        s_up, s_down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_g, ev_f, ev_o, ev_b = (torch.cuda.Event() for _ in range(4))
        first = [True]

        def e2e_step():
            if not first[0]:
                s_up.wait_event(ev_b)               # d_gout free (previous backward done)
                stream.wait_event(ev_o)             # out free (previous download done)
            first[0] = False
            with torch.cuda.stream(s_up):
                d_gout.copy_(h_gout, non_blocking=True)
            ev_g.record(s_up)
            d_ctrl.copy_(h_ctrl, non_blocking=True)
            nb.nurbs_surface_fwd(sh, d_ctrl, U, V, u, v, tables, out, stream)
            ev_f.record(stream)
            s_down.wait_event(ev_f)
            with torch.cuda.stream(s_down):
                h_out.copy_(out, non_blocking=True)
            ev_o.record(s_down)
            stream.wait_event(ev_g)
            if windowed:
                gb.flat.zero_()
            nb.nurbs_surface_bwd(sh, d_ctrl, U, V, u, v, tables, d_gout, g_ctrl, g_U, gb.grad_V, ws,
                                 ws_bytes, stream)
            reduce()
            ev_b.record(stream)
            h_grad.copy_(gb.flat, non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        E = args.e2e_steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(E):
            e2e_step()
        stream.wait_event(ev_o)  # the last download is inside the timed region
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cpu" if share else dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = te.item() / E
        h2d = ctrl.numel() * 4 + gout.numel() * 4
        d2h = out.numel() * 4 + gb.flat.numel() * 4
        e2e = {"value": all_points / (e2e_ms * 1e-3), "unit": "points/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
               "note": "pinned host ctrl+grad_out -> device, fwd+bwd via the C ABI, out+grads -> host; "
                       "dL/dS upload overlapped with the forward and its output download (two copy streams)"}

    # ---------------- oracle cpu baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_grid(args)

    if rank == 0:
        clk = sampler.summary()
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "points/s",
            "n_gpus": world,
            "steps": K,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak" if (args.config == 4 and args.weak) else "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded lattice+N(0,0.1) control nets, U(0.5,1.5) weights, N(0,1) dL/dS)",
            "config": grid_config(args, world),
            "rank0_units": [lo, hi],
            "plan": plan,
            "ctrl_rows": [r0, r1],
            "fwd_points_per_s": fwd_value,
            "fwd_ms": fwd_ms,
            "bwd_ms": bwd_ms,
            "allreduce_ms": red_ms if (world > 1 and args.config == 5) else None,
            "allreduce_bytes": gb.nbytes if args.config == 5 else None,
            "bwd_path": "tcgen05 3xTF32 (--tc)" if args.tc else "SIMT grid kernel",
            "tc_bwd": tc_line,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * K,
            **({"plumbing_only": f"NB_BENCH_SHARE_GPU=1: {world} ranks on {torch.cuda.device_count()} GPU(s) with a "
                                 "gloo group; checks the N-rank launch, sharding and reduction path, the timings are "
                                 "not scaling numbers"} if share else {}),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    args = parse(argv)
    rank, world, local = world_info()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (the driver's own line)
        return subprocess.call(torchrun_cmd(args.gpus, argv))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with --nproc-per-node {args.gpus}")
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.config in (1, 2):
        return run_latency(args, rank, world) if rank == 0 else None
    if args.config == 3:
        return run_fit(args, rank, world) if rank == 0 else None
    if args.derivs:
        return run_derivs(args, rank, world) if rank == 0 else None
    if args.paired:
        return run_paired(args, rank, world)
    if args.knots:
        return run_knots(args, rank, world) if rank == 0 else None
    return run_grid(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main() or 0)
