set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo bench rc=$?
cat gpurun_out/bench_r01.json; tail -3 gpurun_out/bench_r01.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r01.json 2> gpurun_out/bench_ref_r01.err; echo ref rc=$?
cat gpurun_out/bench_ref_r01.json
