set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP_ALGO=ldg5;TK_FP_ALGO=ldg4;TK_FP_ALGO=ldg5,TK_FP2_MINB=12" > gpurun_out/sweep_fp5.log 2>&1; echo sweep rc=$?
head -3 gpurun_out/sweep_fp5.log
timeout 600 python -m pytest tests -m gpu -q -x -k "fp_variants or Golden or smoke or overlapped" > gpurun_out/pytest_gpu7.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu7.log
