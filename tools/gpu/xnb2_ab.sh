#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -k "XNB" > gpurun_out/xnb2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/xnb2_tests.log
tail -3 gpurun_out/xnb2_tests.log
for x in 0 2 1; do for c in C3 C2; do
  NNMG_REG_XNB=$x timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-solve --no-mixed > gpurun_out/xnb2_${c}_$x.json 2> gpurun_out/xnb2_${c}_$x.err
  python - <<PY
import json
d=json.load(open("gpurun_out/xnb2_${c}_$x.json"))
print("$c XNB=$x: fp64", round(d["ms_per_step"],3), "ms vmult", round(d["roofline"]["avg_launch_ms"]*1e3,1), "us frac", round(d["roofline"]["frac"],3))
PY
done; done
