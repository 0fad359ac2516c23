#!/bin/bash
# elasticity apply: TMA-staged geometry slices / block-local nodes A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x -k "ELAST" > gpurun_out/r2_g14_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_g14_tests.log
tail -3 gpurun_out/r2_g14_tests.log
timeout 600 python tools/gpu/elast_variants.py NNMG_ELAST_XCH=1 NNMG_ELAST_BLN=1 NNMG_ELAST_BLN=1,NNMG_ELAST_TMA=1 NNMG_ELAST_XCH=1 NNMG_ELAST_BLN=1 NNMG_ELAST_BLN=1,NNMG_ELAST_TMA=1 2>&1 | tee gpurun_out/r2_g14_elast.txt
