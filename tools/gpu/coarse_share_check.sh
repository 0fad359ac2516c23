#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coarse_direct.py tests/test_gpu_distributed.py -q -x > gpurun_out/r2_g24_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_g24_tests.log
tail -15 gpurun_out/r2_g24_tests.log
