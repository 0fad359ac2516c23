#!/bin/bash
# distributed path: GPU tests + world-1 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split_apply.py tests/test_gpu_distributed.py -q -x > gpurun_out/r2_g13_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_g13_tests.log
tail -4 gpurun_out/r2_g13_tests.log
for c in C3 C5; do
timeout 900 python bench.py --config $c --distributed --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g13_dist_$c.json 2> gpurun_out/r2_g13_dist_$c.err
python - <<PY
import json
d=json.load(open("gpurun_out/r2_g13_dist_$c.json"))
print("$c distributed world 1:", round(d["ms_per_step"],3), "ms", round(d["value"],3), "GDoF/s e2e", round(d["e2e"]["value"],3), "roof", d["roofline"] and round(d["roofline"]["frac"],3))
PY
done
