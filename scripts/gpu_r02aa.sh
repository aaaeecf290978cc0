set -x
mkdir -p gpurun_out
timeout 1200 python scripts/bench_next.py --out gpurun_out/bench_next_aa.json > gpurun_out/bench_next_aa.log 2>&1; echo next rc=$?
cat gpurun_out/bench_next_aa.log | tail -12
