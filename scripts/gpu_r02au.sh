# z-mirror-pair FP with 8-column view tiles vs the default.
set -x
mkdir -p gpurun_out
C="TK_FP_MIRROR=0;TK_FP_MIRROR=1;TK_FP_MIRROR=1,TK_FP_CFG=8x3c8;TK_FP_MIRROR=1,TK_FP_CFG=4x6c8;TK_FP_MIRROR=1,TK_FP_CFG=8x2c8;TK_FP_MIRROR=1,TK_FP_CFG=8x4c8;TK_FP_MIRROR=1,TK_FP_CFG=6x2;TK_FP_MIRROR=0"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_mirror_au.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_mirror_au.log
