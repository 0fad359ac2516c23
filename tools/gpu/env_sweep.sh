# bench one config under several environment settings:
# bash tools/gpu/env_sweep.sh C3 "NNMG_RESTRICT_KERNEL=0 NNMG_RESTRICT_CHUNK=5" "NNMG_RESTRICT_KERNEL=2" ...
c=$1; shift
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/env_${c}_$i.json 2>/dev/null
  echo "[$e] $(python tools/summarize_bench.py gpurun_out/env_${c}_$i.json | cut -d'|' -f3-5)"
done
