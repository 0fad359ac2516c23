#!/bin/bash
# mixed-precision cycle with the fp32-tile coarse solve: tests + bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_coarse_direct.py tests/test_gpu_variants.py tests/test_gpu_parity.py -q -x > gpurun_out/r2_g20_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_g20_tests.log
tail -4 gpurun_out/r2_g20_tests.log
for c in "$@"; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g20_$c.json 2> gpurun_out/r2_g20_$c.err
  python - <<PY
import json
d=json.load(open("gpurun_out/r2_g20_$c.json"))
print("$c: fp64", round(d["ms_per_step"],3), "ms; mixed", round(d["mixed_precision"]["ms_per_step"],3), "ms", round(d["mixed_precision"]["value"],3), "GDoF/s its", d["mixed_precision"]["solve_iterations"], "fp64 its", d["solve"]["iterations"], d["config"]["coarse_solver"])
PY
done
