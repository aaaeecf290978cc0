# FP with the fixed layout's z pitch as an immediate (TK_FP_ZP=1, default) vs the runtime pitch.
set -x
mkdir -p gpurun_out
C="TK_FP_ZP=0;TK_FP_ZP=1;TK_FP_ZP=0;TK_FP_ZP=1"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_zp_az.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_zp_az.log
