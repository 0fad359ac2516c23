#!/bin/bash
# ncu --set full of the fp32 fine-level apply inside one mixed-precision V-cycle
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
c=${1:-C3}
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"${2:-k_apply_reg}" --launch-skip 16 -c 2 -f -o gpurun_out/prof_mixed_$c python tools/gpu/mixed_profile.py $c > gpurun_out/prof_mixed_$c.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_mixed_$c.ncu-rep > gpurun_out/prof_mixed_${c}_summary.txt 2>&1
python tools/ncu_sass_hot.py gpurun_out/prof_mixed_$c.ncu-rep "float" 40 > gpurun_out/prof_mixed_${c}_sass.txt 2>&1
rm -f gpurun_out/prof_mixed_$c.ncu-rep
grep -A3 "float" gpurun_out/prof_mixed_${c}_summary.txt | head -8
