set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP_ALGO=ldg4;TK_FP_ALGO=ldg2;TK_FP_ALGO=ldg4,TK_FP2_MINB=12" > gpurun_out/sweep_fp4.log 2>&1; echo sweep rc=$?
head -3 gpurun_out/sweep_fp4.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu5.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu5.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r02.json')); print(d['value'], d['ms_per_step'], d['kernels'], d['e2e'])"
