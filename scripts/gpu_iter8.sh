set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP_ALGO=mix;TK_FP_ALGO=ldg4" > gpurun_out/sweep_mix.log 2>&1; echo sweep rc=$?
head -2 gpurun_out/sweep_mix.log
timeout 600 python -m pytest tests -m gpu -q -x -k "fp_variants" > gpurun_out/pytest_gpu9.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu9.log
