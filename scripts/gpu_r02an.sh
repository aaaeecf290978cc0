# FP CTA composition A/B: views per CTA x columns per view tile (a warp stays 4 columns x 8 rows of
# one view) and CTA order (o1: view groups fastest).
set -x
mkdir -p gpurun_out
C="TK_FP_CFG=8x2;TK_FP_CFG=16x2c8;TK_FP_CFG=32x2c4;TK_FP_CFG=8x4c8;TK_FP_CFG=4x2c32;TK_FP_CFG=8x2o1;TK_FP_CFG=16x2c8o1;TK_FP_CFG=8x2"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_tiles_an.log 2>&1; echo rc=$?
tail -10 gpurun_out/fp_tiles_an.log
