"""Instruction counts of the bicubic grid kernels in a library (SASS), for A/B of codegen."""
import re, subprocess, sys
lib = sys.argv[1]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, counts = None, {}
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1); counts[cur] = {"n": 0, "FFMA2": 0, "BRA": 0}; continue
    if cur and re.match(r"\s+/\*[0-9a-f]{4,6}\*/", line):
        c = counts[cur]; c["n"] += 1
        for k in ("FFMA2", "BRA"):
            if k in line: c[k] += 1
pat = sys.argv[2] if len(sys.argv) > 2 else r"nurbs_grid_kernelILi3ELi3ELb[01]ELi1ELb0ELb0E"
for k, v in counts.items():
    if re.search(pat, k): print(k[:70], v)
