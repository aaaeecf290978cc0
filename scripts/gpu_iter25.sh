set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_i25.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_i25.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_i25.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke_i25.log
timeout 1200 python bench.py > gpurun_out/bench_i25.json 2> gpurun_out/bench_i25.err; echo bench rc=$?
cat gpurun_out/bench_i25.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cone_|fft_filter|quad|coef" --csv --log-file gpurun_out/launches_i25.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_ncu_i25.log 2>&1; echo ncu rc=$?
