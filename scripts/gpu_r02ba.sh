# FP without the predicated cell move (cell = id every sample), vs the runtime-pitch instance.
set -x
mkdir -p gpurun_out
C="TK_FP_ZP=1;TK_FP_ZP=0;TK_FP_ZP=1;TK_FP_CFG=8x2"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_mf_ba.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_mf_ba.log
