set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_y.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_y.log
timeout 900 python scripts/e2e_breakdown.py > gpurun_out/e2e_y.json 2> gpurun_out/e2e_y.err; echo e2e rc=$?
cat gpurun_out/e2e_y.json; tail -3 gpurun_out/e2e_y.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_y.json 2> gpurun_out/bench_y.err; echo bench rc=$?
python -c "import json; d=json.loads(open('gpurun_out/bench_y.json').read()); print(d['value'], d['ms_per_step'], d['e2e'])"
