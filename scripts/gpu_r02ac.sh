set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ac.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_ac.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ac.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke_ac.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_ac.json 2> gpurun_out/bench_ac.err; echo bench rc=$?
cat gpurun_out/bench_ac.json; tail -3 gpurun_out/bench_ac.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_ac.json 2> gpurun_out/bench_ref_ac.err; echo ref rc=$?
cat gpurun_out/bench_ref_ac.json; tail -3 gpurun_out/bench_ref_ac.err
