#!/bin/bash
# C4 pencil apply: split x launch bound
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "8 0" "8 4" "8 6" "4 2" "4 3"; do
  set -- $v
  NNMG_APPLY_SPLIT=$1 NNMG_APPLY_MINB=$2 timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-solve --no-mixed > gpurun_out/r2_g22.json 2> gpurun_out/r2_g22.err
  python - <<PY
import json
d=json.load(open("gpurun_out/r2_g22.json"))
print("split $1 minb $2: V", round(d["ms_per_step"],3), "ms vmult", round(d["roofline"]["avg_launch_ms"]*1e3,1), "us frac", round(d["roofline"]["frac"],3))
PY
done
