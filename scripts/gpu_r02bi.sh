# Unroll-3 FP default: -m gpu suite, bench, cfg3 timing.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_bi.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_bi.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_bi.json 2> gpurun_out/bench_bi.err; echo bench rc=$?
tail -3 gpurun_out/bench_bi.err
timeout 1200 python scripts/bench_configs.py > gpurun_out/configs_bi.json 2> gpurun_out/configs_bi.err; echo configs rc=$?
