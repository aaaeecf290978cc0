set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 300 python -m pytest tests -m gpu -q -x -k "slab" > gpurun_out/pytest_i23.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_i23.log
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP_ALGO=ldg4m;TK_FP_ALGO=slab" > gpurun_out/sweep_fp23.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_fp23.log
TK_FP_ALGO=slab timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cone_fp_slab" -c 1 -o gpurun_out/prof_slab python scripts/prof_step.py --what fp > gpurun_out/ncu_slab.log 2>&1; echo ncu rc=$?
