# Re-entry validation after the container re-creation: full -m gpu suite, smoke, bench, reference arm.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_al.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_al.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_al.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke_al.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_al.json 2> gpurun_out/bench_al.err; echo bench rc=$?
cat gpurun_out/bench_al.json; tail -3 gpurun_out/bench_al.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_al.json 2> gpurun_out/bench_ref_al.err; echo ref rc=$?
cat gpurun_out/bench_ref_al.json; tail -3 gpurun_out/bench_ref_al.err
