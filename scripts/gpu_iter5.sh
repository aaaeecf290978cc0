set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu6.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu6.log
timeout 900 python scripts/fp_sweep.py --op bp --configs "TK_BP_ALGO=smem;TK_BP_ALGO=quad" > gpurun_out/sweep_bp.log 2>&1; echo sweep rc=$?
head -2 gpurun_out/sweep_bp.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r03.json 2> gpurun_out/bench_r03.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r03.json')); print(d['value'], d['ms_per_step'], d['kernels'], d['e2e'])"
tail -3 gpurun_out/bench_r03.err
