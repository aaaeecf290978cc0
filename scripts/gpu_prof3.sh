set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
TK_BP_ALGO=smem timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cone_bp_smem|fft_filter" -c 2 -o gpurun_out/prof_r05 python scripts/prof_step.py --views 120 --what fdk > gpurun_out/ncu5.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu5.log
