set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python scripts/bench_variants.py --fp ldg2 --bp quad,ldg --reps 2 --out gpurun_out/variants_r03.json > gpurun_out/variants3.log 2>&1; echo variants rc=$?
cat gpurun_out/variants3.log | tail -4
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu3.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cone_fp2_kernel|cone_bp_quad_kernel|fft_filter_kernel|quadify" -s 1 -c 4 -o gpurun_out/prof_r03 python scripts/prof_step.py > gpurun_out/ncu3.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu3.log
