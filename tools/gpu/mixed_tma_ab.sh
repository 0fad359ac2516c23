#!/bin/bash
# fp32 register apply: whole-chunk TMA staging of the geometry (NNMG_REG_TMA=1) A/B on the mixed C3 cycle
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NNMG_REG_TMA=1 timeout 900 python -m pytest tests/test_gpu_mixed.py -q -x -k "C3 or C1 or graph" > gpurun_out/mixed_tma_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/mixed_tma_tests.log
tail -3 gpurun_out/mixed_tma_tests.log
for t in 0 1; do
  NNMG_REG_TMA=$t timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/mixed_tma_$t.json 2> gpurun_out/mixed_tma_$t.err
  python - <<PY
import json
d=json.load(open("gpurun_out/mixed_tma_$t.json"))
print("REG_TMA=$t: fp64", round(d["ms_per_step"],3), "ms; mixed", round(d["mixed_precision"]["ms_per_step"],3), "ms", round(d["mixed_precision"]["value"],3))
PY
done
