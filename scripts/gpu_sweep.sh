set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python scripts/fp_sweep.py --op fp --configs "TK_FP2_RAYS=1,TK_FP2_MINB=10;TK_FP2_RAYS=1,TK_FP2_MINB=12;TK_FP2_RAYS=1,TK_FP2_MINB=16;TK_FP2_RAYS=2,TK_FP2_MINB=6;TK_FP2_RAYS=2,TK_FP2_MINB=8;TK_FP2_RAYS=2,TK_FP2_MINB=12" > gpurun_out/sweep_fp.log 2>&1; echo sweep rc=$?
cat gpurun_out/sweep_fp.log
TK_FP2_RAYS=2 timeout 600 python -m pytest tests -m gpu -q -x -k "fp_variants or Golden or cone_fp_bp_64" > gpurun_out/pytest_fp2r.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_fp2r.log
