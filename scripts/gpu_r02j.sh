set -x
mkdir -p gpurun_out
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "TK_FP_MIRROR=0;TK_FP_MIRROR=1;TK_FP_MIRROR=1,TK_FP_CFG=8x1;TK_FP_MIRROR=1,TK_FP_CFG=6x2;TK_FP_MIRROR=0,TK_FP_CFG=4x4" > gpurun_out/fp_sweep_j.log 2>&1; echo sweep rc=$?
cat gpurun_out/fp_sweep_j.log
timeout 900 python scripts/fp_sweep.py --op bp --reps 3 --configs "TK_BP_ALGO=tma;TK_BP_ALGO=quad" > gpurun_out/bp_sweep_j.log 2>&1; echo bp rc=$?
cat gpurun_out/bp_sweep_j.log
