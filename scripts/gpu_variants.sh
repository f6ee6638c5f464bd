#!/bin/bash
# Bench each experiment variant (exp/lib_*.so) on configs 4 and 5.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for so in exp/lib_*.so; do
  v=$(basename $so .so)
  for cfg in 4 5; do
    NURBS_B200_LIB_EXPERIMENT=$PWD/$so timeout 300 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/var_${v}_cfg${cfg}.log 2>&1
    python - "$v" "$cfg" <<'PY'
import json,sys
v,c=sys.argv[1],sys.argv[2]
try:
    l=[x for x in open(f"gpurun_out/var_{v}_cfg{c}.log") if x.startswith("{")][-1]
    d=json.loads(l); print(f"{v:>12} cfg{c} value {d['value']:.3e} fwd {d['fwd_ms']:.4f} bwd {d['bwd_ms']:.4f} fwdfrac {d['roofline']['fwd']['frac']:.3f} bwdfrac {d['roofline']['bwd']['frac']:.3f}")
except Exception as e: print(v,c,"failed",e)
PY
  done
done
