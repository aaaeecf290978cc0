# Slab-staged forward kernel: bit-identity tests, then cfg4 timing against the general kernel.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "Slab or fp_variants" > gpurun_out/pytest_slab_h.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_slab_h.log
timeout 900 python scripts/fp_sweep.py --op fp --reps 3 --configs "TK_FP_SLAB=0;TK_FP_SLAB=1;TK_FP_SLAB=1,TK_FP_T=4;TK_FP_SLAB=1,TK_FP_T=6;TK_FP_SLAB=1,TK_FP_T=12;TK_FP_SLAB=1,TK_FP_SLAB_VG=4;TK_FP_SLAB=1,TK_FP_SLAB_VG=4,TK_FP_T=4" > gpurun_out/fp_sweep_h.log 2>&1; echo sweep rc=$?
cat gpurun_out/fp_sweep_h.log
