set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_i21.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_i21.log
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP_ALGO=ldg4m;TK_FP_ALGO=ldg4d;TK_FP_ALGO=ldg4d,TK_FP2_MINB=10" > gpurun_out/sweep_fp21.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_fp21.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cone_fp4d" -c 1 -o gpurun_out/prof_fp4d python scripts/prof_step.py --what fp > gpurun_out/ncu_fp4d.log 2>&1; echo ncu rc=$?
