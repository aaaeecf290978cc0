# Bench + launch list + full ncu captures of the z-fastest forward projector and the quad-scatter transpose.
set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1200 python bench.py > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err; echo bench rc=$?
cat gpurun_out/bench_k.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cone_|coef_|quad|fft_|pad|crop" -c 200 --csv --log-file gpurun_out/launches_k.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_ncu_k.log 2>&1; echo ncu rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cone_fp4z_kernel|coef_volume_z" -c 2 -o gpurun_out/prof_fp_k python scripts/prof_step.py --what fp > gpurun_out/ncu_fp_k.log 2>&1; echo ncufull rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cone_fp_adjoint4z|unquad_z" -c 2 -o gpurun_out/prof_fpt_k python scripts/grad_bench.py --n 256 --views 180 --det 512 > gpurun_out/ncu_fpt_k.log 2>&1; echo ncufpt rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cone_bp_tma|fft_filter" -c 2 -o gpurun_out/prof_bp_k python scripts/prof_step.py --what fdk > gpurun_out/ncu_bp_k.log 2>&1; echo ncubp rc=$?
timeout 600 python scripts/fp_angle.py > gpurun_out/fp_angle_k.json 2>&1
timeout 600 python scripts/grad_bench.py > gpurun_out/grad_k.json 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_k.json 2> gpurun_out/bench_ref_k.err; echo ref rc=$?
