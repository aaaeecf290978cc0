# FP cell-load flavours: LDG.E.128.CONSTANT (default) vs coherent LDG.E.128 (probe 4) vs the
# LTC256B (L2 256-byte sector-promotion) hint (probe 5).
set -x
mkdir -p gpurun_out
C="TK_FP_PROBE=0;TK_FP_PROBE=4;TK_FP_PROBE=5;TK_FP_PROBE=0;TK_FP_PROBE=5"
timeout 900 python scripts/fp_sweep.py --op fp --reps 2 --configs "$C" > gpurun_out/fp_ld_bj.log 2>&1; echo rc=$?
grep "^fp" gpurun_out/fp_ld_bj.log
