#!/bin/bash
# ncu --set full of the C5 elasticity apply variants: bash tools/gpu/prof_elast.sh "NNMG_ELAST_BLN=1" tag
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
combo="$1"; tag="$2"
timeout 600 python tools/gpu/elast_variants.py $combo > gpurun_out/prof_elast_$tag.plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_apply_reg_elast --launch-skip 10 -c 2 -f \
   -o gpurun_out/prof_elast_$tag python tools/gpu/elast_variants.py $combo > gpurun_out/prof_elast_$tag.ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_elast_$tag.ncu-rep > gpurun_out/prof_elast_${tag}_summary.txt 2>&1
python tools/ncu_sass_hot.py gpurun_out/prof_elast_$tag.ncu-rep "" 40 > gpurun_out/prof_elast_${tag}_sass.txt 2>&1
ncu -i gpurun_out/prof_elast_$tag.ncu-rep --page raw --csv > gpurun_out/prof_elast_${tag}_raw.csv 2>/dev/null
rm -f gpurun_out/prof_elast_$tag.ncu-rep
cat gpurun_out/prof_elast_${tag}_summary.txt
