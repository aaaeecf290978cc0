# Final-ish verification + ncu captures of the default kernels at cfg4.
set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_f1.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_f1.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_f1.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke_f1.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cone_fp4|cone_bp_tma|fft_filter_r16|quad_volume" -c 4 -o gpurun_out/prof_f1 python scripts/prof_step.py > gpurun_out/ncu_f1.log 2>&1; echo ncu rc=$?
