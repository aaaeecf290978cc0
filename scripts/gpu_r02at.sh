# FP z-pair march (two samples' z axis as one packed FFMA2 / FADD2.RM / FADD2 chain) vs default.
set -x
mkdir -p gpurun_out
C="TK_FP_PROBE=0;TK_FP_PROBE=3;TK_FP_PROBE=0;TK_FP_PROBE=3"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_zpair_at.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_zpair_at.log
