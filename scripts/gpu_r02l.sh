# Compile-time-pitch TMA back projector, 2D B^T, warp-cooperative FP A/B, reference suites, BP ncu.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_l.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu_l.log
timeout 300 python scripts/fp_sweep.py --op bp --reps 3 --configs "TK_BP_ALGO=tma;TK_BP_ALGO=quad" > gpurun_out/bp_sweep_l.log 2>&1; echo bp rc=$?
cat gpurun_out/bp_sweep_l.log
timeout 600 python scripts/fp_sweep.py --op fp --reps 2 --configs "TK_FP_ALGO=default;TK_FP_ALGO=warp;TK_FP_ALGO=tex" > gpurun_out/fp_sweep_l.log 2>&1; echo fp rc=$?
cat gpurun_out/fp_sweep_l.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"cone_bp_tma_kernel" -c 1 -o gpurun_out/prof_bp_l python scripts/prof_step.py --what fdk > gpurun_out/ncu_bp_l.log 2>&1; echo ncu rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_l.csv python scripts/prof_step.py --what fp,fdk > gpurun_out/launches_l.log 2>&1; echo launches rc=$?
timeout 600 python scripts/run_reference_suite.py --out gpurun_out/reference_suite_l.json > gpurun_out/refsuite_l.log 2>&1; echo refsuite rc=$?
tail -2 gpurun_out/refsuite_l.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err; echo bench rc=$?
cat gpurun_out/bench_l.json
