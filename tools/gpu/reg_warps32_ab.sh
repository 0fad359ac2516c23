#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do for w in 4 1 2; do
  NNMG_REG_WARPS32=$w timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/rw32_$w.json 2> gpurun_out/rw32_$w.err
  python - <<PY
import json
d=json.load(open("gpurun_out/rw32_$w.json"))
print("C3 REG_WARPS32=$w: fp64", round(d["ms_per_step"],3), "ms | mixed", round(d["mixed_precision"]["ms_per_step"],4), "ms")
PY
done; done
