#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for mb in 2 3 4; do
  NNMG_REG_MINB=$mb timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/r2_g18_mb$mb.json 2> gpurun_out/r2_g18_mb$mb.err
  python - <<PY
import json
d=json.load(open("gpurun_out/r2_g18_mb$mb.json"))
print("MINB $mb: fp64", round(d["ms_per_step"],3), "ms; mixed", d["mixed_precision"]["ms_per_step"], "ms", d["mixed_precision"]["value"])
PY
done
