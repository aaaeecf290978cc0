set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python scripts/bench_variants.py --fp ldg2 --bp quad --reps 2 > gpurun_out/variants4.log 2>&1; echo variants rc=$?
head -2 gpurun_out/variants4.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu4.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu4.log
