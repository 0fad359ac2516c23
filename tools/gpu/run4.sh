#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_determinism.py -q -x > gpurun_out/r2_g4_det.log 2>&1
echo "rc=$?" >> gpurun_out/r2_g4_det.log
timeout 600 python tools/gpu/mixed_profile.py C3 > gpurun_out/r2_g4_mp.log 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_g4_mixed_launches_C3.csv python tools/gpu/mixed_profile.py C3 > gpurun_out/r2_g4_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2_g4_ncu.log
