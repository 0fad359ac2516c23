# restriction chunk sweep: bash tools/gpu/chunk_sweep.sh C3 "1 4 10 20"
c=$1; shift
for ch in $1; do
  NNMG_RESTRICT_CHUNK=$ch timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sw_${c}_$ch.json 2>/dev/null
  echo "chunk $ch: $(python tools/summarize_bench.py gpurun_out/sw_${c}_$ch.json | grep -o 'res [^|]*')"
done
