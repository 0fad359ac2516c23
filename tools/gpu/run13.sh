#!/bin/bash
# split apply / overlap / transfer timing rows: new GPU tests + world-1 distributed bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split_apply.py tests/test_gpu_distributed.py tests/test_gpu_parity.py -q -x > gpurun_out/r2_g13_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_g13_tests.log
for c in C3 C5; do
timeout 900 python bench.py --config $c --distributed --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g13_dist_$c.json 2> gpurun_out/r2_g13_dist_$c.err
done
tail -5 gpurun_out/r2_g13_tests.log
cat gpurun_out/r2_g13_dist_C3.json | cut -c1-600
tail -3 gpurun_out/r2_g13_dist_C3.err
