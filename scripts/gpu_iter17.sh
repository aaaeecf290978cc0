set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 120 python scripts/tma_smoke.py > gpurun_out/tma_smoke.log 2>&1; echo tma rc=$?
cat gpurun_out/tma_smoke.log | tail -3
timeout 600 python -m pytest tests -m gpu -q -x -k "bp or fdk or Golden or smoke" > gpurun_out/pytest_i17.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_i17.log
timeout 600 python scripts/fp_sweep.py --op bp --reps 3 --configs "TK_BP_ALGO=quad;TK_BP_ALGO=tma" > gpurun_out/sweep_bp17.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_bp17.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cone_bp_tma" -c 1 -o gpurun_out/prof_bptma python scripts/prof_step.py --what fdk > gpurun_out/ncu_bptma.log 2>&1; echo ncu rc=$?
