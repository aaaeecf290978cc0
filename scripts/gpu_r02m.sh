set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fp_variants or 2d_bp_transpose or tuning" > gpurun_out/pytest_m.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_m.log
timeout 300 python scripts/fp_sweep.py --op fp --reps 3 --configs "TK_FP_TR=8;TK_FP_TR=16;TK_FP_TR=8" > gpurun_out/fp_sweep_m.log 2>&1; echo fp rc=$?
cat gpurun_out/fp_sweep_m.log
