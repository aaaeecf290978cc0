set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests -m gpu -q -x -k "bp or fdk or Golden or smoke or overlapped or helical" > gpurun_out/pytest_i24.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_i24.log
timeout 600 python scripts/fp_sweep.py --op bp --reps 3 --configs "TK_BP_ZB=16;TK_BP_ZB=32;TK_BP_ALGO=quad" > gpurun_out/sweep_bp24.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_bp24.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cone_bp_tma" -c 1 -o gpurun_out/prof_bptma3 python scripts/prof_step.py --what fdk > gpurun_out/ncu_bptma3.log 2>&1; echo ncu rc=$?
