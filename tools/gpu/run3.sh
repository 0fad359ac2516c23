#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mixed.py -q -x > gpurun_out/r2_g3_mixed.log 2>&1
echo "rc=$?" >> gpurun_out/r2_g3_mixed.log
for c in C3 C5 C2 C4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g3_bench_$c.json 2> gpurun_out/r2_g3_bench_$c.err
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2_g3_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_g3_tests.log
