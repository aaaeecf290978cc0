# FP march unroll factor A/B (1 / 2 default / 3 / 4).
set -x
mkdir -p gpurun_out
C="TK_FP_UNR=2;TK_FP_UNR=1;TK_FP_UNR=3;TK_FP_UNR=4;TK_FP_UNR=2"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_unr_bg.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_unr_bg.log
