#!/bin/bash
# prolongation / lane restriction: warps per CTA
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NNMG_TRANSFER_WARPS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_mixed.py -q -x -k "transfer or restrict or prolong or mixed" > gpurun_out/tw_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/tw_tests.log
tail -3 gpurun_out/tw_tests.log
for c in C3 C5 C2; do for w in 4 2 1; do
  NNMG_TRANSFER_WARPS=$w timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-solve --no-mixed > gpurun_out/tw_$w.json 2> gpurun_out/tw_$w.err
  python - <<PY
import json
d=json.load(open("gpurun_out/tw_$w.json")); k=d["kernels"]
print("$c TRANSFER_WARPS=$w: V", round(d["ms_per_step"],3), "ms pro", round(k["prolongate_ms"]*1e3,1), "us", round(k["prolongate_roof_frac"],3), "res", round(k["restrict_ms"]*1e3,1), "us", round(k["restrict_roof_frac"],3))
PY
done; done
