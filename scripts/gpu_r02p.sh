set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "transpose or matched or adjoint or determin" > gpurun_out/pytest_p.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_p.log
timeout 900 python scripts/fpt_sweep.py --configs "TK_FPT_SEG=1;TK_FPT_SEG=2;TK_FPT_SEG=3;TK_FPT_SEG=4;TK_FPT_SEG=6;DET=1,TK_FPT_SEG=1;DET=1,TK_FPT_SEG=3" > gpurun_out/fpt_sweep_p.log 2>&1; echo sweep rc=$?
cat gpurun_out/fpt_sweep_p.log
