# FP with an L2 prefetch (prefetch.global.L2) of the cell rows PF samples ahead, once per 8 samples.
set -x
mkdir -p gpurun_out
C="TK_FP_PF=0;TK_FP_PF=8;TK_FP_PF=16;TK_FP_PF=32;TK_FP_PF=0"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_pf_bf.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_pf_bf.log
