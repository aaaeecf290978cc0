set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests -m gpu -q -x -k "Golden or fdk or overlapped or fbp or filter" > gpurun_out/pytest_gpu13.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu13.log
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP2_MINB=10;TK_FP2_MINB=12" > gpurun_out/sweep_fp6.log 2>&1; echo sweep rc=$?
head -2 gpurun_out/sweep_fp6.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r07.json 2> gpurun_out/bench_r07.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r07.json')); print(d['value'], d['ms_per_step'], d['kernels'], d['e2e'])"
