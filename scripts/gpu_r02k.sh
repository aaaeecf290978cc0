# After the library prune: whole GPU suite, racecheck of the TMA back projector, the reference's own
# suites on libtkb200, a fresh ncu capture of the default forward kernel, launch list, bench, reference arm.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_k.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu_k.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool racecheck --racecheck-report all --print-limit 20 python scripts/sanitize_cases.py bp filter > gpurun_out/san_racecheck_k.log 2>&1; echo racecheck rc=$?
tail -3 gpurun_out/san_racecheck_k.log
timeout 1500 python scripts/run_reference_suite.py --out gpurun_out/reference_suite_k.json > gpurun_out/refsuite_k.log 2>&1; echo refsuite rc=$?
tail -3 gpurun_out/refsuite_k.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"cone_fp_kernel" -c 1 -o gpurun_out/prof_fp_k python scripts/prof_step.py --what fp > gpurun_out/ncu_fp_k.log 2>&1; echo ncu rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_k.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/bench_ncu_k.log 2>&1; echo launches rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err; echo bench rc=$?
cat gpurun_out/bench_k.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_k.json 2> gpurun_out/bench_ref_k.err; echo ref rc=$?
cat gpurun_out/bench_ref_k.json
