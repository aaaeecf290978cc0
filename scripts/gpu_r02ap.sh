# 8x2 vs 8x4c8 FP launch (repeated A/B), ncu of the back projector (per-view constants in the
# parameter block) and of the row filter.
set -x
mkdir -p gpurun_out
C="TK_FP_CFG=8x2;TK_FP_CFG=8x4c8;TK_FP_CFG=8x2;TK_FP_CFG=8x4c8;TK_FP_CFG=8x2;TK_FP_CFG=8x4c8"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_ab_ap.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_ab_ap.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"cone_bp_tma_kernel" -c 1 -o gpurun_out/prof_bp_ap python scripts/prof_step.py --what fdk > gpurun_out/ncu_bp_ap.log 2>&1; echo ncu rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fft_filter" -c 1 -o gpurun_out/prof_filt_ap python scripts/prof_step.py --what fdk > gpurun_out/ncu_filt_ap.log 2>&1; echo ncu rc=$?
