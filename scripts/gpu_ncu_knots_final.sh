#!/bin/bash
# ncu evidence of the knot-gradient call: launch lists (configs 4 and 5) and one --set full
# capture of each mode's grid kernel (config 4: per-row weights, config 5: span moments).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/knf; mkdir -p $O
for c in 4 5; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_cfg$c.csv python bench.py --knots --config $c --steps 3 --warmup 3 > /dev/null 2>&1
  ncu --set full --clock-control none -k regex:nurbs_grid_kernel -s 3 -c 1 -f -o $O/prof_cfg$c python bench.py --knots --config $c --steps 2 --warmup 3 > /dev/null 2>&1
done
ls -la $O
python scripts/ncu_summary.py --tag r02_knots_cfg4 --cfg knots4 --launches $O/launches_cfg4.csv --full $O/prof_cfg4.ncu-rep > /dev/null 2>&1
python scripts/ncu_summary.py --tag r02_knots_cfg5 --cfg knots5 --launches $O/launches_cfg5.csv --full $O/prof_cfg5.ncu-rep > /dev/null 2>&1
mkdir -p gpurun_out/knf_out; cp profiles/r02_knots_cfg*_summary.txt profiles/r02_knots_cfg*_launches.csv profiles/ncu_traffic.json gpurun_out/knf_out/ 2>/dev/null
rm -f $O/*.ncu-rep
