#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coarse_direct.py tests/test_gpu_determinism.py -q -x > gpurun_out/coarse_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/coarse_tests.log
tail -3 gpurun_out/coarse_tests.log
timeout 900 python tools/gpu/coarse_direct_bench.py 2>&1 | tail -6
for c in C2 C5; do
timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-solve --no-mixed > gpurun_out/coarse_$c.json 2>/dev/null
python tools/summarize_bench.py gpurun_out/coarse_$c.json | cut -c1-60
done
