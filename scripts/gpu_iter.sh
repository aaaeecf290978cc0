set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python scripts/bench_variants.py --fp ldg2,tex --bp ldg --reps 2 --out gpurun_out/variants_r02.json > gpurun_out/variants2.log 2>&1; echo variants rc=$?
cat gpurun_out/variants2.log | tail -4
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_ldg2.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu_ldg2.log
