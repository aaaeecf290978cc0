set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_q.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu_q.log
grep -E "SKIP|skipped" gpurun_out/pytest_gpu_q.log | head -5
timeout 300 python scripts/fp_sweep.py --op fp --reps 3 --configs "TK_FP_MIRROR=0" > gpurun_out/fp_q.log 2>&1; echo fp rc=$?
cat gpurun_out/fp_q.log
