set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python scripts/bench_variants.py --out gpurun_out/variants_r01.json > gpurun_out/variants.log 2>&1; echo variants rc=$?
cat gpurun_out/variants.log | tail -8
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_texfp.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_texfp.log
TK_BP_ALGO=tex timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_texbp.log 2>&1; echo pytest-texbp rc=$?
tail -3 gpurun_out/pytest_gpu_texbp.log
