set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "determin or transpose" > gpurun_out/pytest_u.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|Error|assert" gpurun_out/pytest_u.log | head -10
timeout 600 python scripts/fpt_sweep.py --configs "TK_FPT_CARRY=1;DET=1" > gpurun_out/fpt_u.log 2>&1; echo sweep rc=$?
cat gpurun_out/fpt_u.log
