# Upload-ordered row-band FP pipeline: GPU tests, e2e breakdown (rows vs views), bench.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py -q -x > gpurun_out/pytest_pipe_av.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_pipe_av.log
for m in rows views rows; do
TK_FP_PIPE=$m timeout 600 python scripts/e2e_breakdown.py > gpurun_out/e2e_${m}_av.json 2>gpurun_out/e2e_${m}_av.err; echo "$m rc=$?"; cat gpurun_out/e2e_${m}_av.json; tail -2 gpurun_out/e2e_${m}_av.err
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_av.json 2> gpurun_out/bench_av.err; echo bench rc=$?
tail -c 1500 gpurun_out/bench_av.json | head -c 400; tail -3 gpurun_out/bench_av.err
