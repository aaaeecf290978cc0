set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "fixed_row or Cfg3 or tuning or fp_variants" > gpurun_out/pytest_w.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_w.log
timeout 900 python scripts/bench_configs.py > gpurun_out/configs_w.json 2> gpurun_out/configs_w.err; echo configs rc=$?
cat gpurun_out/configs_w.json
