#!/bin/bash
# ncu launch list (kernel times) of one V-cycle + hot kernels: bash tools/gpu/launches.sh C2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
c=${1:-C2}
timeout 600 python bench.py --config $c --profile --no-cpu-baseline > gpurun_out/plain_$c.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_$c.csv python bench.py --config $c --profile --no-cpu-baseline > gpurun_out/ncu_l_$c.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$c.csv | head -50
