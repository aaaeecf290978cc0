# 8-column 8x4 FP default: full -m gpu suite, bench, launch list, ncu of the FP kernel.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_aq.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_aq.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_aq.json 2> gpurun_out/bench_aq.err; echo bench rc=$?
cat gpurun_out/bench_aq.json; tail -3 gpurun_out/bench_aq.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_aq.csv python scripts/prof_step.py --what fp,fdk > gpurun_out/launches_aq.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cone_fp_kernel" -c 1 -o gpurun_out/prof_fp_aq python scripts/prof_step.py --what fp > gpurun_out/ncu_fp_aq.log 2>&1; echo ncu rc=$?
