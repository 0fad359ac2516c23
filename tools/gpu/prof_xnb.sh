#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export NNMG_REG_XNB=1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off --nvtx --nvtx-include "hot/" \
     -k regex:'k_apply_reg' -c 1 -f -o gpurun_out/prof_xnb python bench.py --config C3 --profile --no-cpu-baseline > gpurun_out/ncu_xnb.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_xnb.ncu-rep > gpurun_out/prof_xnb_summary.txt 2>&1
python tools/ncu_sass_hot.py gpurun_out/prof_xnb.ncu-rep "" 30 > gpurun_out/prof_xnb_sass.txt 2>&1
rm -f gpurun_out/prof_xnb.ncu-rep
cat gpurun_out/prof_xnb_summary.txt
