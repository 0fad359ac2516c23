#!/bin/bash
# C5 transfer sweep: restriction chunk x work-item size
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for mp in 0 96 64; do for ch in 0 2 3 4; do
  export -n NNMG_TRANSFER_MAXP NNMG_RESTRICT_CHUNK; unset NNMG_TRANSFER_MAXP NNMG_RESTRICT_CHUNK
  [ $mp != 0 ] && export NNMG_TRANSFER_MAXP=$mp
  [ $ch != 0 ] && export NNMG_RESTRICT_CHUNK=$ch
  timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-solve --no-mixed > gpurun_out/r2_g19.json 2> gpurun_out/r2_g19.err
  python - <<PY
import json
d=json.load(open("gpurun_out/r2_g19.json"))
k=d["kernels"]
print("maxp $mp chunk $ch: V", round(d["ms_per_step"],3), "ms pro", round(k["prolongate_ms"]*1e3,1), "us res", round(k["restrict_ms"]*1e3,1), "us")
PY
done; done
