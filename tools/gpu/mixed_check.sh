#!/bin/bash
# mixed-precision cycle with single-precision arithmetic: tests + bench of the given configs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mixed.py -q -x -s > gpurun_out/r2_g17_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_g17_tests.log
grep "mixed vs\|passed\|failed\|rc=\|Error\|assert" gpurun_out/r2_g17_tests.log | tail -16
for a in 32 64; do for c in "$@"; do
  NNMG_MIXED_ARITH=$a timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g17_${c}_a$a.json 2> gpurun_out/r2_g17_${c}_a$a.err
  python - <<PY
import json
d=json.load(open("gpurun_out/r2_g17_${c}_a$a.json"))
print("$c arith $a: fp64", round(d["ms_per_step"],3), "ms; mixed", d["mixed_precision"]["ms_per_step"], "ms", d["mixed_precision"]["value"], "GDoF/s its", d["mixed_precision"]["solve_iterations"], "fp64 its", d["solve"]["iterations"])
PY
done; done
