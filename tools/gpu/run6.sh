#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --target-processes all python tools/gpu/sanitize.py > gpurun_out/r2_sanitizer_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/r2_sanitizer_$tool.log
done
