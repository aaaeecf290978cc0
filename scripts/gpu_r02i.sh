set -x
mkdir -p gpurun_out
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "TK_FP_SLAB=0;TK_FP_SLAB=1;TK_FP_SLAB=1,TK_FP_SLAB_DIAG=1;TK_FP_SLAB=1,TK_FP_T=4,TK_FP_SLAB_DIAG=1;TK_FP_SLAB=1,TK_FP_T=16,TK_FP_SLAB_DIAG=1;TK_FP_SLAB=1,TK_FP_SLAB_CAP=1024;TK_FP_SLAB=1,TK_FP_T=16;TK_FP_SLAB=1,TK_FP_T=24" > gpurun_out/fp_sweep_i.log 2>&1; echo sweep rc=$?
cat gpurun_out/fp_sweep_i.log
