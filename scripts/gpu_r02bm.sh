# Final closing records: bench + reference arm, launch list, ncu of the FP, cfg1-3, cfg5 gradient, smoke.
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_bm.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke_bm.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_bm.json 2> gpurun_out/bench_bm.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_bm.json 2> gpurun_out/bench_ref_bm.err; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bm.csv python scripts/prof_step.py --what fp,fdk > gpurun_out/launches_bm.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cone_fp_kernel" -c 1 -o gpurun_out/prof_fp_bm python scripts/prof_step.py --what fp > gpurun_out/ncu_fp_bm.log 2>&1; echo ncu rc=$?
timeout 1200 python scripts/bench_configs.py > gpurun_out/configs_bm.json 2> gpurun_out/configs_bm.err; echo configs rc=$?
timeout 900 python scripts/grad_bench.py > gpurun_out/grad_bm.json 2> gpurun_out/grad_bm.err; echo grad rc=$?
