set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests -m gpu -q -x -k "fp_variants or Golden or fdk" > gpurun_out/pytest_i22.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_i22.log
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP_ALGO=ldg4m;TK_FP_ALGO=ldg4p;TK_FP_ALGO=ldg4p,TK_FP2_MINB=10" > gpurun_out/sweep_fp22.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_fp22.log
TK_FP_ALGO=ldg4p TK_FP2_MINB=10 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cone_fp4p" -c 1 -o gpurun_out/prof_fp4p python scripts/prof_step.py --what fp > gpurun_out/ncu_fp4p.log 2>&1; echo ncu rc=$?
