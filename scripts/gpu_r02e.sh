# Round 2 re-entry box: whole GPU suite, compute-sanitizer on small cases,
# mirror vs z-fastest FP at cfg4, the reference's own suites on libtkb200, bench.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_e.log 2>&1; echo pytest rc=$?
tail -8 gpurun_out/pytest_gpu_e.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check no --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/san_memcheck_e.log 2>&1; echo memcheck rc=$?
tail -4 gpurun_out/san_memcheck_e.log
timeout 900 $CS --tool racecheck --racecheck-report all --print-limit 50 python scripts/sanitize_cases.py bp filter > gpurun_out/san_racecheck_e.log 2>&1; echo racecheck rc=$?
tail -4 gpurun_out/san_racecheck_e.log
timeout 900 $CS --tool synccheck --print-limit 50 python scripts/sanitize_cases.py bp filter fp > gpurun_out/san_synccheck_e.log 2>&1; echo synccheck rc=$?
tail -4 gpurun_out/san_synccheck_e.log
timeout 600 python scripts/fp_band_probe.py --rows 128 1024 > gpurun_out/fp_band_e.log 2>&1; echo probe rc=$?
cat gpurun_out/fp_band_e.log
timeout 1500 python scripts/run_reference_suite.py --out gpurun_out/reference_suite_e.json > gpurun_out/refsuite_e.log 2>&1; echo refsuite rc=$?
tail -3 gpurun_out/refsuite_e.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; echo bench rc=$?
cat gpurun_out/bench_e.json; tail -3 gpurun_out/bench_e.err
