#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/gpu/coarse_direct_bench.py > gpurun_out/r2_coarse_direct.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2_g2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_g2_tests.log
for c in C4 C5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g2_bench_$c.json 2> gpurun_out/r2_g2_bench_$c.err
done
