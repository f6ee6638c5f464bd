"""Per-source-line instruction and stall attribution of one kernel in an ncu report.

ncu's SASS page gives (address, instructions executed, stall samples) per instruction; a
cubin of the same build disassembled with `nvdisasm -gi` maps each SASS offset to a source
line. Usage:
    python scripts/sass_lines.py <report.ncu-rep> <cubin> <mangled-kernel> [kernel-regex]
Prints the top source lines by executed warp instructions, with stall-sample shares.
"""
import collections, csv, io, re, subprocess, sys

rep, cubin, mangled = sys.argv[1:4]
kre = sys.argv[4] if len(sys.argv) > 4 else "."
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for ln in src.splitlines():
    if ln.startswith('"Kernel Name"'):
        cur = [ln]; blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
prof = None
for b in blocks:
    if re.search(kre, b[0]):
        prof = b; break
rr = list(csv.reader(io.StringIO("\n".join(prof[1:]))))
h = rr[0]; ix = {k: i for i, k in enumerate(h)}
rows = []
for r in rr[1:]:
    if len(r) < len(h): continue
    rows.append((int(r[ix["Address"]], 16), int(r[ix["Instructions Executed"]] or 0),
                 int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r[ix["Source"]].strip()))
base = rows[0][0]
sass = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
lines = sass.splitlines()
start = None
for k, ln in enumerate(lines):
    if ln.startswith(".text." + mangled + ":"):
        start = k; break
# nvdisasm prints the inline chain innermost first, then the outer call sites; key = the
# innermost line plus the call site one level inside the kernel body (MODE=inner|outer|both)
import os
MODE = os.environ.get("MODE", "both")
off2line, curline, chain = {}, "?", []
for ln in lines[start + 1:]:
    if ln.startswith(".text.") or ln.startswith("//-----"):
        break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
    if m:
        chain.append(f"{m.group(1).split('/')[-1].replace('nurbs_', '').replace('.cuh', '')}:{m.group(2)}")
        inner, outer = chain[0], (chain[-2] if len(chain) > 1 else chain[-1])
        curline = {"inner": inner, "outer": outer}.get(MODE, inner if inner == outer else f"{inner}@{outer}")
        continue
    chain = []
    m = re.match(r"\s*/\*([0-9a-f]{4,6})\*/\s+(.*?)\s*;?\s*$", ln)
    if m:
        off2line[int(m.group(1), 16)] = (curline, m.group(2))
tot = sum(r[1] for r in rows) or 1
stot = sum(r[2] for r in rows) or 1
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
mism = 0
for a, n, st, s in rows:
    line, txt = off2line.get(a - base, ("?", ""))
    if txt.split()[:1] != s.split()[:1]:
        mism += 1
    agg[line][0] += n; agg[line][1] += st
    t = s.split(); op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "")).split(".")[0]
    agg[line][2][op] += n
print(f"instructions {tot}  stall samples {stot}  sass/cubin opcode mismatches {mism} of {len(rows)}")
for line, (n, st, ops) in sorted(agg.items(), key=lambda x: -x[1][0])[:int(sys.argv[5]) if len(sys.argv) > 5 else 45]:
    print(f"{line:24s} {n:11d} {n/tot:6.3f}  stall {st/stot:6.3f}  " + " ".join(f"{k}:{v//max(1,min(ops.values()))}" for k, v in ops.most_common(5)))
