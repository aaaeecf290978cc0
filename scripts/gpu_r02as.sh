# FP roofline decomposition: the access stream alone (probe 1) and the arithmetic alone (probe 2)
# against the projector, plus ncu of both probes.
set -x
mkdir -p gpurun_out
C="TK_FP_PROBE=0;TK_FP_PROBE=1;TK_FP_PROBE=2;TK_FP_PROBE=0"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_probe_as.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_probe_as.log
for pr in 1 2; do
TK_FP_PROBE=$pr timeout 900 ncu --set full --clock-control none -k regex:"cone_fp_kernel" -c 1 -o gpurun_out/prof_fp_probe${pr}_as python scripts/prof_step.py --what fp > gpurun_out/ncu_fp_probe${pr}_as.log 2>&1; echo ncu rc=$?
done
