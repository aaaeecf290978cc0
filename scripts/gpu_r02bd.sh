# Matched A^T occupancy A/B at cfg5: 8 (48 regs, 40 warps/SM), 12 (40 regs), 16 (32 regs) CTAs per SM.
set -x
mkdir -p gpurun_out
timeout 900 python scripts/fpt_sweep.py --configs "TK_FPT_MINB=8;TK_FPT_MINB=12;TK_FPT_MINB=16;TK_FPT_MINB=8" > gpurun_out/fpt_minb_bd.log 2>&1; echo rc=$?
grep "^TK" gpurun_out/fpt_minb_bd.log
