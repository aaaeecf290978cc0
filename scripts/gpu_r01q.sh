# Bench + launch list + full ncu captures of the z-fastest forward projector and the quad-scatter transpose.
set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1200 python bench.py > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
cat gpurun_out/bench_q.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cone_|coef_|quad|fft_|pad|crop" -c 200 --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_ncu_q.log 2>&1; echo ncu rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cone_fp4z_kernel|coef_volume_z" -c 2 -o gpurun_out/prof_fp_q python scripts/prof_step.py --what fp > gpurun_out/ncu_fp_q.log 2>&1; echo ncufull rc=$?
timeout 600 python scripts/fp_angle.py > gpurun_out/fp_angle_q.json 2>&1
timeout 600 python scripts/grad_bench.py > gpurun_out/grad_q.json 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_q.json 2> gpurun_out/bench_ref_q.err; echo ref rc=$?
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_q.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_q.log 2>&1; echo pytest rc=$?
