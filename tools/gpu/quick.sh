# quick check: GPU tests, then bench lines (no CPU baseline) for the given configs
# usage: bash tools/gpu/quick.sh C3 C4 C5
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in "$@"; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err; echo "$c rc=$?"
  python tools/summarize_bench.py gpurun_out/q_$c.json 2>/dev/null
done
