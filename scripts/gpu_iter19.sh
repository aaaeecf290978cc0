set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_i19.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_i19.log
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP_ALGO=ldg4m;TK_FP_ALGO=ldg4" > gpurun_out/sweep_fp19.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_fp19.log
timeout 600 python scripts/fp_sweep.py --op bp --reps 3 --configs "TK_BP_ALGO=quad;TK_BP_ALGO=tma" > gpurun_out/sweep_bp19.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_bp19.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/bench_i19.json 2> gpurun_out/bench_i19.err; echo bench rc=$?
cat gpurun_out/bench_i19.json
