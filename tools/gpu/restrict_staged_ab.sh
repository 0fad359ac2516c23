#!/bin/bash
# staged restriction (C4, C5): reduction buffer aliased onto the staging buffers, launch bound
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_mixed.py -q -x -k "transfer or restrict or mixed" > gpurun_out/rs_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/rs_tests.log
tail -3 gpurun_out/rs_tests.log
for c in C4 C5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/rs_$c.json 2> gpurun_out/rs_$c.err
  python - <<PY
import json
d=json.load(open("gpurun_out/rs_$c.json")); k=d["kernels"]
print("$c: V", round(d["ms_per_step"],3), "ms mixed", round(d["mixed_precision"]["ms_per_step"],3), "pro", round(k["prolongate_ms"]*1e3,1), "us res", round(k["restrict_ms"]*1e3,1), "us", round(k["restrict_roof_frac"],3))
PY
done
