set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tuning" > gpurun_out/pytest_s.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_s.log
timeout 600 python scripts/fp_sweep.py --op fp --reps 3 --configs "TK_FP_PF=0;TK_FP_PF=1;TK_FP_PF=4;TK_FP_PF=6;TK_FP_PF=10;TK_FP_PF=0" > gpurun_out/fp_s.log 2>&1; echo fp rc=$?
cat gpurun_out/fp_s.log
