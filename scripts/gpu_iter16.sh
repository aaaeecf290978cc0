set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_i16.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_i16.log
timeout 600 python scripts/fp_sweep.py --op filter --reps 5 --configs "TK_FILTER_ALGO=stockham;TK_FILTER_ALGO=r16" > gpurun_out/sweep_filt16.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_filt16.log
timeout 900 python scripts/fp_sweep.py --op bp --reps 3 --configs "TK_BP_ALGO=quad;TK_BP_ALGO=quad,TK_BP_Q42=1" > gpurun_out/sweep_bp16.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_bp16.log
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP_ALGO=ldg4m;TK_FP_ALGO=ldg4" > gpurun_out/sweep_fp16.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_fp16.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fft_filter_r16" -c 1 -o gpurun_out/prof_filt3 python scripts/prof_step.py --what fdk > gpurun_out/ncu_filt3.log 2>&1; echo ncu rc=$?
