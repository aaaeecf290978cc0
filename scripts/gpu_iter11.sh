set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests -m gpu -q -x -k "bp_variants or bp_row_band or Golden or Oracle or overlapped" > gpurun_out/pytest_gpu12.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu12.log
grep -E "Error|assert" gpurun_out/pytest_gpu12.log | head -5
timeout 900 python scripts/fp_sweep.py --op bp --configs "TK_BP_ALGO=pairs;TK_BP_ALGO=quad" > gpurun_out/sweep_bp2.log 2>&1; echo sweep rc=$?
head -2 gpurun_out/sweep_bp2.log
