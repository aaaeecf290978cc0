set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests -m gpu -q -x -k "cone or smoke or Golden" > gpurun_out/pytest_fp8.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_fp8.log
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP_ALGO=ldg4;TK_FP_ALGO=ldg8;TK_FP_ALGO=ldg8,TK_FP2_MINB=10;TK_FP_ALGO=ldg8,TK_FP2_MINB=8" > gpurun_out/sweep_fp8.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_fp8.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cone_fp8" -c 1 -o gpurun_out/prof_fp8 python scripts/prof_step.py --what fp > gpurun_out/ncu_fp8.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_fp8.log
