# Bench + launch list + full ncu capture of the forward projector (per-ray orientation copy).
set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1200 python bench.py > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err; echo bench rc=$?
cat gpurun_out/bench_i.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_i.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_ncu_i.log 2>&1; echo ncu rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cone_fp4_kernel" -c 1 -o gpurun_out/prof_fp_i python scripts/prof_step.py --what fp > gpurun_out/ncu_fp_i.log 2>&1; echo ncufull rc=$?
tail -3 gpurun_out/ncu_fp_i.log
