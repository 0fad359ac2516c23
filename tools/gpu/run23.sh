#!/bin/bash
# launch list of the world-size-1 distributed cycle (C3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config C3 --distributed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dist_plain.json 2> gpurun_out/dist_plain.err || { tail -5 gpurun_out/dist_plain.err; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --launch-skip 2000 --launch-count 400 \
   --log-file gpurun_out/launches_dist_C3.csv python bench.py --config C3 --distributed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dist_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/launches_dist_C3.csv | head -40
cut -c1-200 gpurun_out/dist_plain.json
