#!/bin/bash
# staged restriction: planes per lane A/B on C4 / C5 (+ elasticity apply default check)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -k "planes_per_lane or ELAST" > gpurun_out/r2_g15_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_g15_tests.log
tail -3 gpurun_out/r2_g15_tests.log
for pl in 1 2; do for c in C4 C5; do
  NNMG_RESTRICT_PL=$pl timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g15_${c}_pl$pl.json 2> gpurun_out/r2_g15_${c}_pl$pl.err
  echo "PL=$pl $(python tools/summarize_bench.py gpurun_out/r2_g15_${c}_pl$pl.json | cut -c1-150)"
done; done
