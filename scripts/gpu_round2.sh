# Round check after the r16 filter / Q42 BP / ldg4m FP defaults.
set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_r2.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_r2.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke_r2.log
timeout 1200 python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench rc=$?
cat gpurun_out/bench_r2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cone_|fft_filter|quad|coef" --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_ncu_r2.log 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cone_fp4|cone_bp_quad|fft_filter_r16|quadify|quad_volume" -c 5 -o gpurun_out/prof_r2 python scripts/prof_step.py > gpurun_out/ncu_r2.log 2>&1; echo ncu rc=$?
