"""Summarise an ncu --set full report of one kernel: key metrics, instruction mix, and the
instructions grouped by execution count (loop nests) with their stall samples.
Usage: python scripts/sass_hot.py <report.ncu-rep> [kernel-regex]"""
import csv, collections, io, re, subprocess, sys
rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if not re.search(kre, d.get("Kernel Name", "")): continue
    print(d.get("Kernel Name", "")[:90])
    for k in keys:
        if k in d: print(f"  {k} = {d[k]}")
    st = {k: d[k] for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    top = sorted(st.items(), key=lambda x: -float(x[1] or 0))[:8]
    print("  stalls:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]} {float(v):.2f}" for k, v in top))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
lines = src.splitlines()
# one kernel per block: header line then column names
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]; blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
for b in blocks:
    if not re.search(kre, b[0]): continue
    rr = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    h = rr[0]; ix = {k: i for i, k in enumerate(h)}
    data = []
    for r in rr[1:]:
        if len(r) < len(h): continue
        try: n = int(r[ix["Instructions Executed"]] or 0)
        except ValueError: continue
        data.append((n, int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r[ix["Source"]]))
    tot = sum(x[0] for x in data); sst = sum(x[1] for x in data) or 1
    ops = collections.Counter()
    for n, _, s_ in data:
        t = s_.split(); op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "")).split(".")[0]; ops[op] += n
    print("  instructions", tot, "top ops:", ", ".join(f"{k} {v/tot:.3f}" for k, v in ops.most_common(14)))
    g = collections.defaultdict(lambda: [0, 0, 0])
    for n, st_, _ in data:
        g[n][0] += n; g[n][1] += st_; g[n][2] += 1
    for n, (t, st_, c) in sorted(g.items(), key=lambda x: -x[1][0])[:14]:
        print(f"  exec/instr {n:9d} x {c:5d} instr = {t:11d} ({t/tot:.3f})  stall samples {st_/sst:.3f}")
