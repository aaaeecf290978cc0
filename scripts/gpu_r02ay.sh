# Row filter with packed complex arithmetic (FADD2/FMUL2/FFMA2): timing at cfg4 and the filter parity tests.
set -x
mkdir -p gpurun_out
timeout 600 python scripts/fp_sweep.py --op filter --reps 5 --configs "A=1;A=2" > gpurun_out/filt_ay.log 2>&1; echo rc=$?
grep "^filter" gpurun_out/filt_ay.log
timeout 900 python -m pytest tests -m gpu -q -x -k "filter or fdk or fbp or cfg" > gpurun_out/pytest_filt_ay.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_filt_ay.log
