set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cone_fp4_kernel|cone_bp_quad_kernel|fft_filter_kernel" -s 1 -c 3 -o gpurun_out/prof_r04 python scripts/prof_step.py > gpurun_out/ncu4.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu4.log
