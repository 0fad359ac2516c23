#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/gpu/apply_modes.py C3 C4 C5 C2 > gpurun_out/r2_apply_modes.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_coarse_stress.py -q -x > gpurun_out/r2_g8_stress.log 2>&1
echo "rc=$?" >> gpurun_out/r2_g8_stress.log
