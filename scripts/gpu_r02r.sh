set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fp_variants or tuning" > gpurun_out/pytest_r.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_r.log
timeout 300 python scripts/fp_sweep.py --op fp --reps 3 --configs "TK_FP_XMAP=0;TK_FP_XMAP=1;TK_FP_XMAP=0;TK_FP_XMAP=1" > gpurun_out/fp_r.log 2>&1; echo fp rc=$?
cat gpurun_out/fp_r.log
