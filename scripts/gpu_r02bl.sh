# Ray set-up with one fp64 division per clip axis and rsqrt normalisation: FP timing, whole -m gpu suite.
set -x
mkdir -p gpurun_out
timeout 900 python scripts/fp_sweep.py --op fp --reps 3 --configs "TK_FP_PROBE=0;TK_FP_PROBE=7;TK_FP_PROBE=0" > gpurun_out/fp_setup_bl.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_setup_bl.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_bl.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_bl.log
