#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box, from gpurun_out/ files).

    python scripts/ncu_summary.py --tag r01_cfg4 --cfg 4 --launches gpurun_out/launches_X.csv \
        --full gpurun_out/prof_X.ncu-rep

Writes profiles/<tag>_launches.csv (the per-launch list, cleaned), profiles/<tag>_summary.txt
(duration, DRAM bytes, issue / occupancy, stall reasons per captured kernel, the kernel's share
of the step from the launch list) and updates profiles/ncu_traffic.json with the measured
dram__bytes_read.sum + dram__bytes_write.sum per launch (bench.py's roofline "traffic").
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    name = name.replace("nb::", "")
    return name.split("(")[0] if "(nb::Params" in name or "(Params" in name else name[:60]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--cfg", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full")
    a = ap.parse_args()
    out_dir = os.path.join(ROOT, "profiles")
    os.makedirs(out_dir, exist_ok=True)
    lines = []
    if a.launches:
        txt = open(a.launches).read()
        body = txt[txt.index('"ID"'):]
        rows = list(csv.DictReader(io.StringIO(body)))
        with open(os.path.join(out_dir, f"{a.tag}_launches.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["id", "kernel", "grid", "block", "gpu__time_duration_ns"])
            for r in rows:
                w.writerow([r["ID"], short(r["Kernel Name"]), r["Grid Size"], r["Block Size"], r["Metric Value"]])
        agg = collections.OrderedDict()
        for r in rows:
            agg.setdefault(short(r["Kernel Name"]), []).append(float(r["Metric Value"]))
        lines.append("== launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised)")
        steady = {k: v for k, v in agg.items() if "grid_kernel" in k}
        tot = sum(sum(v[3:]) / max(1, len(v[3:])) for v in steady.values()) if steady else 0
        for k, v in agg.items():
            vv = v[3:] if len(v) > 3 else v
            avg = sum(vv) / len(vv)
            share = f"  share of step {100 * avg / tot:5.1f}%" if k in steady and tot else ""
            lines.append(f"  {k:<45} launches {len(v):>3}  avg {avg / 1e3:9.2f} us{share}")
    if a.full:
        raw = subprocess.run(["ncu", "-i", a.full, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        traffic_path = os.path.join(out_dir, "ncu_traffic.json")
        traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
        lines.append("\n== ncu --set full (one launch each)")
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            name = short(d["Kernel Name"])
            def mb(k):
                v = float(d[k])
                return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u[k], 1.0)
            rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
            lines.append(f"  {name}")
            lines.append(f"    duration {float(d['gpu__time_duration.sum']):.2f} {u['gpu__time_duration.sum']}"
                         f"   dram read {rd:.1f} MB  write {wr:.1f} MB  ({d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']}% of peak dram)")
            lines.append(f"    instructions {float(d['smsp__inst_executed.sum']) / 1e6:.1f} M   issue {d['sm__inst_executed.sum.pct_of_peak_sustained_elapsed']}%"
                         f"   warps active {d['sm__warps_active.avg.pct_of_peak_sustained_active']}%   regs {d['launch__registers_per_thread']}"
                         f"   smem/block {d['launch__shared_mem_per_block_dynamic']} {u['launch__shared_mem_per_block_dynamic']}")
            st = [(k.split("stalled_")[1].split("_per")[0], float(d[k])) for k in hdr
                  if "warps_issue_stalled" in k and k.endswith("per_issue_active.ratio") and d[k]]
            st = sorted([x for x in st if x[1] > 0.1], key=lambda x: -x[1])
            lines.append("    stalls per issue: " + ", ".join(f"{k} {v:.2f}" for k, v in st))
            kn = d["Kernel Name"]
            if "<" not in kn:  # untemplated helper kernels (reduce, validate): no traffic entry
                continue
            targs = kn.split("<", 1)[1].split(">", 1)[0].replace("(int)", "").replace("(bool)", "")
            targs = [x.strip() for x in targs.split(",")]
            if "points_" in kn:
                kind = "bwd" if "bwd" in kn else "fwd"
            else:
                kind = "bwd" if len(targs) > 2 and targs[2] in ("1", "true") else "fwd"  # <P, Q, BWD, ...>
            traffic.setdefault(f"cfg{a.cfg}", {})[kind] = {"kernel": name, "dram_bytes_per_launch": (rd + wr) * 1e6,
                                                          "source": os.path.basename(a.full), "tag": a.tag}
        json.dump(traffic, open(traffic_path, "w"), indent=1)
    text = "\n".join(lines) + "\n"
    open(os.path.join(out_dir, f"{a.tag}_summary.txt"), "w").write(text)
    print(text)


if __name__ == "__main__":
    main()
