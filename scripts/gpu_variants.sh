#!/bin/bash
# Bench each experiment variant (exp/lib_*.so) on configs 4 and 5 (kernel-only lines).
# VARIANT_ENVS="NAME=ENV=VAL ..." adds runs of every lib with an extra environment variable.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() {  # $1 tag, $2 lib, $3 cfg, rest: env
  local tag=$1 so=$2 cfg=$3; shift 3
  env "$@" NURBS_B200_LIB_EXPERIMENT=$PWD/$so timeout 300 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/var_${tag}_cfg${cfg}.log 2>&1
  python - "$tag" "$cfg" <<'PY'
import json,sys
v,c=sys.argv[1],sys.argv[2]
try:
    l=[x for x in open(f"gpurun_out/var_{v}_cfg{c}.log") if x.startswith("{")][-1]
    d=json.loads(l); print(f"{v:>16} cfg{c} value {d['value']:.3e} fwd {d['fwd_ms']:.4f} bwd {d['bwd_ms']:.4f} fwdfrac {d['roofline']['fwd']['frac']:.3f} bwdfrac {d['roofline']['bwd']['frac']:.3f}")
except Exception as e: print(v,c,"failed",e)
PY
}
for so in exp/lib_*.so; do
  v=$(basename $so .so)
  for cfg in ${CFGS:-4 5}; do
    run $v $so $cfg NB_DUMMY=1
    for ve in ${VARIANT_ENVS}; do run "${v}_${ve%%=*}" $so $cfg "${ve#*=}"; done
  done
done
