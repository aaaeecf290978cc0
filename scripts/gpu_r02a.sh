# Round 2, first box: new full-size config parity tests, the whole GPU suite,
# bench (ours + the tomokit reference arm), and the 2-rank code path (gloo, one GPU).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt
timeout 1200 python -m pytest tests/test_gpu_configs.py -m gpu -q -rA > gpurun_out/pytest_cfg_a.log 2>&1; echo cfg rc=$?
tail -25 gpurun_out/pytest_cfg_a.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo bench rc=$?
cat gpurun_out/bench_a.json; tail -5 gpurun_out/bench_a.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_a.json 2> gpurun_out/bench_ref_a.err; echo ref rc=$?
cat gpurun_out/bench_ref_a.json; tail -5 gpurun_out/bench_ref_a.err
TK_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 1 --warmup 1 --no-e2e > gpurun_out/bench_gloo2_a.json 2> gpurun_out/bench_gloo2_a.err; echo gloo2 rc=$?
cat gpurun_out/bench_gloo2_a.json; tail -5 gpurun_out/bench_gloo2_a.err
TK_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --fdk angle --steps 1 --warmup 1 --no-e2e > gpurun_out/bench_gloo2b_a.json 2> gpurun_out/bench_gloo2b_a.err; echo gloo2b rc=$?
cat gpurun_out/bench_gloo2b_a.json; tail -5 gpurun_out/bench_gloo2b_a.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_a.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu_a.log
