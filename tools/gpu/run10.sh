#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/gpu/elast_variants.py > gpurun_out/r2_elast_xch.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k "C4" > gpurun_out/r2_g9_full_C4.log 2>&1
echo "rc=$?" >> gpurun_out/r2_g9_full_C4.log
