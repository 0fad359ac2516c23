#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_g12_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_g12_tests.log
timeout 600 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g12_bench_C5.json 2> gpurun_out/r2_g12_bench_C5.err
