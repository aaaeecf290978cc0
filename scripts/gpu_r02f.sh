# Ray segments x kernel (general / mirror) x launch configuration at cfg4, then the GPU suite.
set -x
mkdir -p gpurun_out
timeout 900 python scripts/fp_sweep.py --op fp --reps 3 --configs "TK_FP_MIRROR=0;TK_FP_MIRROR=0,TK_FP_SEG=2;TK_FP_MIRROR=0,TK_FP_SEG=3;TK_FP_MIRROR=0,TK_FP_SEG=4;TK_FP_MIRROR=1;TK_FP_MIRROR=1,TK_FP_SEG=2;TK_FP_MIRROR=1,TK_FP_SEG=3;TK_FP_MIRROR=1,TK_FP_SEG=4;TK_FP_MIRROR=1,TK_FP_SEG=2,TK_FP_CFG=8x1;TK_FP_MIRROR=1,TK_FP_SEG=3,TK_FP_CFG=8x1;TK_FP_MIRROR=1,TK_FP_SEG=2,TK_FP_CFG=8x2;TK_FP_MIRROR=0,TK_FP_SEG=2,TK_FP_CFG=4x4;TK_FP_MIRROR=1,TK_FP_SEG=6" > gpurun_out/fp_sweep_f.log 2>&1; echo sweep rc=$?
cat gpurun_out/fp_sweep_f.log
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu_f.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu_f.log
