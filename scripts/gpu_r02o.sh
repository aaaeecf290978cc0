set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "transpose or matched or adjoint or determin" > gpurun_out/pytest_o.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_o.log
timeout 600 python scripts/fpt_sweep.py --configs "TK_FPT_CARRY=1;TK_FPT_CARRY=0;DET=1" > gpurun_out/fpt_sweep_o.log 2>&1; echo sweep rc=$?
cat gpurun_out/fpt_sweep_o.log
