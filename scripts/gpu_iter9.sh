set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu10.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu10.log
grep -E "Error|assert|FAILED" gpurun_out/pytest_gpu10.log | head -5
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r05.json 2> gpurun_out/bench_r05.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r05.json')); print(d['value'], d['ms_per_step'], d['kernels'], d['e2e'])"
