# Round-2 record: GPU suite, smoke, bench (ours + reference arm), launch list.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_t.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_t.log 2>&1; echo smoke rc=$?
cat gpurun_out/smoke_t.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err; echo bench rc=$?
cat gpurun_out/bench_t.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_t.json 2> gpurun_out/bench_ref_t.err; echo ref rc=$?
cat gpurun_out/bench_ref_t.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_t.csv python scripts/prof_step.py --what fp,fdk > gpurun_out/launches_t.log 2>&1; echo launches rc=$?
