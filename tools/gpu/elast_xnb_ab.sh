#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NNMG_ELAST_XNB=1 timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_mixed.py tests/test_gpu_parity.py -q -x -k "el or C5 or ELAST" > gpurun_out/exnb_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/exnb_tests.log
tail -3 gpurun_out/exnb_tests.log
timeout 600 python tools/gpu/elast_variants.py NNMG_ELAST_XNB=0 NNMG_ELAST_XNB=1 NNMG_ELAST_XNB=0 NNMG_ELAST_XNB=1
for x in 0 1; do
  NNMG_ELAST_XNB=$x timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/exnb_$x.json 2> gpurun_out/exnb_$x.err
  python - <<PY
import json
d=json.load(open("gpurun_out/exnb_$x.json"))
print("C5 ELAST_XNB=$x: fp64", round(d["ms_per_step"],3), "ms vmult", round(d["roofline"]["avg_launch_ms"]*1e3,1), "us frac", round(d["roofline"]["frac"],3), "| mixed", round(d["mixed_precision"]["ms_per_step"],3), "ms")
PY
done
