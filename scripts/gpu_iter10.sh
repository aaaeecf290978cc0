set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests -m gpu -q -x -k "fp_variants or Golden or Oracle or overlapped" > gpurun_out/pytest_gpu11.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu11.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r06.json 2> gpurun_out/bench_r06.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r06.json')); print(d['value'], d['ms_per_step'], d['kernels'], d['e2e'])"
