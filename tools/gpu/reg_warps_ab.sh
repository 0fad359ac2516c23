#!/bin/bash
# fp64 register Laplace apply: warps (cell blocks) per CTA
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do for c in C3 C2; do for w in 4 1 2; do
  NNMG_REG_WARPS=$w timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-solve --no-mixed > gpurun_out/rw_$w.json 2> gpurun_out/rw_$w.err
  python - <<PY
import json
d=json.load(open("gpurun_out/rw_$w.json"))
print("$c REG_WARPS=$w: fp64", round(d["ms_per_step"],4), "ms vmult", round(d["roofline"]["avg_launch_ms"]*1e3,2), "us frac", round(d["roofline"]["frac"],3))
PY
done; done; done
