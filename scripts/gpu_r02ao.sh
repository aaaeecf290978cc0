# FP dual cell layout (y-row and x-row copies, each ray on the copy whose row axis is its major
# horizontal axis) with (TK_FP_DUAL=1) and without (=2) the lead/trail row carry-over.
set -x
mkdir -p gpurun_out
C="TK_FP_DUAL=0;TK_FP_DUAL=1;TK_FP_DUAL=1,TK_FP_CFG=4x3;TK_FP_DUAL=1,TK_FP_CFG=6x2;TK_FP_DUAL=1,TK_FP_CFG=8x4c8;TK_FP_DUAL=2,TK_FP_CFG=8x2;TK_FP_DUAL=2,TK_FP_CFG=4x3;TK_FP_DUAL=0,TK_FP_CFG=8x4c8;TK_FP_DUAL=0,TK_FP_CFG=8x2"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_dual_ao.log 2>&1; echo rc=$?
tail -12 gpurun_out/fp_dual_ao.log
