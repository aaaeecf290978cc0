set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python scripts/prof_step.py --reps 2 > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cone_fp_kernel|cone_bp_kernel|fft_filter_kernel" -s 1 -c 3 -o gpurun_out/prof_r01 python scripts/prof_step.py > gpurun_out/ncu_full.log 2>&1; echo ncufull rc=$?
tail -5 gpurun_out/ncu_full.log
