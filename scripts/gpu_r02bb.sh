# Round-2 closing records: whole -m gpu suite, smoke, sanitizers on the changed kernels, bench + reference
# arm, launch list, ncu of the default FP, other BASELINE configs, cfg5 gradient, reference suites.
set -x
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_bb.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_bb.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_bb.log 2>&1; echo smoke rc=$?
tail -2 gpurun_out/smoke_bb.log
timeout 900 $CS --tool memcheck --leak-check no --print-limit 50 python scripts/sanitize_cases.py fp bp > gpurun_out/san_memcheck_bb.log 2>&1; echo memcheck rc=$?
tail -3 gpurun_out/san_memcheck_bb.log
timeout 900 $CS --tool racecheck --racecheck-report all --print-limit 50 python scripts/sanitize_cases.py bp > gpurun_out/san_racecheck_bb.log 2>&1; echo racecheck rc=$?
tail -3 gpurun_out/san_racecheck_bb.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_bb.json 2> gpurun_out/bench_bb.err; echo bench rc=$?
tail -3 gpurun_out/bench_bb.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_bb.json 2> gpurun_out/bench_ref_bb.err; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bb.csv python scripts/prof_step.py --what fp,fdk > gpurun_out/launches_bb.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cone_fp_kernel" -c 1 -o gpurun_out/prof_fp_bb python scripts/prof_step.py --what fp > gpurun_out/ncu_fp_bb.log 2>&1; echo ncu rc=$?
timeout 1200 python scripts/bench_configs.py > gpurun_out/configs_bb.json 2> gpurun_out/configs_bb.err; echo configs rc=$?
timeout 900 python scripts/grad_bench.py > gpurun_out/grad_bb.json 2> gpurun_out/grad_bb.err; echo grad rc=$?
timeout 1500 python scripts/run_reference_suite.py --out gpurun_out/reference_suite_bb.json > gpurun_out/refsuite_bb.log 2>&1; echo refsuite rc=$?
tail -2 gpurun_out/refsuite_bb.log
