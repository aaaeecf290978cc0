set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_i26.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_i26.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quad|fft|cone" -c 4 --csv --log-file gpurun_out/launches_i26.csv python scripts/prof_step.py --what fp > gpurun_out/b_ncu_i26.log 2>&1; echo ncu rc=$?
cat gpurun_out/launches_i26.csv | grep -i quad | cut -c1-200
