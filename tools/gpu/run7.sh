#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/gpu/dual_sweep.py C3 > gpurun_out/r2_dual_sweep.txt 2>&1
