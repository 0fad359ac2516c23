#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(time timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -x) > gpurun_out/fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/fullsize.log
tail -8 gpurun_out/fullsize.log
