# FP unroll 3 vs 2, repeated.
set -x
mkdir -p gpurun_out
C="TK_FP_UNR=2;TK_FP_UNR=3;TK_FP_UNR=2;TK_FP_UNR=3;TK_FP_UNR=2;TK_FP_UNR=3"
timeout 900 python scripts/fp_sweep.py --op fp --reps 3 --configs "$C" > gpurun_out/fp_unr_bh.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_unr_bh.log
