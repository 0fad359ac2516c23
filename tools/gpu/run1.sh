#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_g1_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_g1_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_g1_tests.log
for c in C2 C5 C4 C3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g1_bench_$c.json 2> gpurun_out/r2_g1_bench_$c.err
done
