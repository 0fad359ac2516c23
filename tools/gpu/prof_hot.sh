# ncu --set full of the isolated fine-level hot kernels (NVTX range hot/) for the given configs
# usage: bash tools/gpu/prof_hot.sh '<kernel regex>' C3 C4 ...
re="$1"; shift
for c in "$@"; do
  timeout 600 python bench.py --config $c --profile --no-cpu-baseline > gpurun_out/plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off --nvtx --nvtx-include "hot/" \
     -k regex:"$re" -c 4 -f -o gpurun_out/prof_$c python bench.py --config $c --profile --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1
  echo "$c prof rc=$?"
done
