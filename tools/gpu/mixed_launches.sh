#!/bin/bash
# launch list of one fp64 and one mixed-precision V-cycle (C3), kernel times by ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
c=${1:-C3}
timeout 600 python tools/gpu/mixed_profile.py $c > gpurun_out/mixed_plain_$c.log 2>&1 || { tail -5 gpurun_out/mixed_plain_$c.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/launches_mixed_$c.csv python tools/gpu/mixed_profile.py $c > gpurun_out/mixed_ncu_$c.log 2>&1
python tools/launch_summary.py gpurun_out/launches_mixed_$c.csv | head -60
