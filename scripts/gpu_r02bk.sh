# Closing records for the final code (unroll-3 FP): smoke, bench + reference arm, launch list,
# ncu of the default FP kernel, cfg5 gradient, memcheck of the FP cases.
set -x
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_bk.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke_bk.log
timeout 900 $CS --tool memcheck --leak-check no --print-limit 50 python scripts/sanitize_cases.py fp > gpurun_out/san_memcheck_bk.log 2>&1; echo memcheck rc=$?
tail -1 gpurun_out/san_memcheck_bk.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_bk.json 2> gpurun_out/bench_bk.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_bk.json 2> gpurun_out/bench_ref_bk.err; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bk.csv python scripts/prof_step.py --what fp,fdk > gpurun_out/launches_bk.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cone_fp_kernel" -c 1 -o gpurun_out/prof_fp_bk python scripts/prof_step.py --what fp > gpurun_out/ncu_fp_bk.log 2>&1; echo ncu rc=$?
timeout 900 python scripts/grad_bench.py > gpurun_out/grad_bk.json 2> gpurun_out/grad_bk.err; echo grad rc=$?
