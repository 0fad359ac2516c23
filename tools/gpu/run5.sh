#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k "not C4" > gpurun_out/r2_g5_full.log 2>&1
echo "rc=$?" >> gpurun_out/r2_g5_full.log
