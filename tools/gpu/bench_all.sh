#!/bin/bash
# bench lines for every config + the reference arm (-> tools/update_profiles.py rN)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in C3 C4 C5 C2 C1; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?"
