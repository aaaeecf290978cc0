set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_i13.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_i13.log
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP_ALGO=ldg4;TK_FP_ALGO=ldg4m;TK_FP_ALGO=ldg4m,TK_FP2_MINB=10" > gpurun_out/sweep_fp13.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_fp13.log
timeout 900 python scripts/fp_sweep.py --op bp --reps 3 --configs "TK_BP_ALGO=quad;TK_BP_ALGO=coef" > gpurun_out/sweep_bp13.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_bp13.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cone_bp_coef" -c 1 -o gpurun_out/prof_bpcoef python scripts/prof_step.py --what fdk > gpurun_out/ncu_bp.log 2>&1; echo ncu rc=$?
TK_FP_ALGO=ldg4m timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cone_fp4" -c 1 -o gpurun_out/prof_fp4m python scripts/prof_step.py --what fp > gpurun_out/ncu_fp4m.log 2>&1; echo ncu rc=$?
