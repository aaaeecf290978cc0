set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q -x -k "filter or fp_variants or Golden or fdk" > gpurun_out/pytest_i15.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_i15.log
timeout 600 python scripts/fp_sweep.py --op filter --reps 5 --configs "TK_FILTER_ALGO=stockham;TK_FILTER_ALGO=r16" > gpurun_out/sweep_filt15.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_filt15.log
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP_ALGO=ldg4m;TK_FP_ALGO=ldg4m,TK_FP_WR=4;TK_FP_ALGO=ldg4m,TK_FP_WR=8" > gpurun_out/sweep_fp15.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_fp15.log
TK_FP_WR=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cone_fp4" -c 1 -o gpurun_out/prof_fp4wr8 python scripts/prof_step.py --what fp > gpurun_out/ncu_fpwr.log 2>&1; echo ncu rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fft_filter_r16" -c 1 -o gpurun_out/prof_filt2 python scripts/prof_step.py --what fdk > gpurun_out/ncu_filt2.log 2>&1; echo ncu rc=$?
