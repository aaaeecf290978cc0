# FP CTA size around the 8x4c8 optimum (views x CTAs/SM x columns per view tile).
set -x
mkdir -p gpurun_out
C="TK_FP_CFG=8x4c8;TK_FP_CFG=4x8c8;TK_FP_CFG=8x8c4;TK_FP_CFG=16x4c4;TK_FP_CFG=2x8c16;TK_FP_CFG=4x16c4;TK_FP_CFG=8x4c8"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_cta_ar.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_cta_ar.log
