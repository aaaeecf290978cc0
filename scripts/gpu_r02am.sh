# FP software-pipelined march A/B: P = next sample's cell loaded right after the current
# interpolation (one buffer), Q = two-deep (two buffers), at several occupancies.
set -x
mkdir -p gpurun_out
C="TK_FP_CFG=8x2;TK_FP_CFG=8x2P;TK_FP_CFG=4x4P;TK_FP_CFG=6x2;TK_FP_CFG=6x2P;TK_FP_CFG=4x3P;TK_FP_CFG=5x2P;TK_FP_CFG=8x1P;TK_FP_CFG=5x2Q;TK_FP_CFG=4x2Q;TK_FP_CFG=8x1Q;TK_FP_CFG=4x3Q;TK_FP_CFG=8x2"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_pipe_am.log 2>&1; echo rc=$?
cat gpurun_out/fp_pipe_am.log | tail -16
