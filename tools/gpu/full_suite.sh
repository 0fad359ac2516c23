#!/bin/bash
# full GPU suite + smoke at HEAD
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(time timeout 2400 python -m pytest tests -m gpu -q) > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -6 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
