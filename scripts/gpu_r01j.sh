# Bench + launch list + full ncu captures of the z-fastest forward projector and the quad-scatter transpose.
set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1200 python bench.py > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err; echo bench rc=$?
cat gpurun_out/bench_j.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_j.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_ncu_j.log 2>&1; echo ncu rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cone_fp4z_kernel|quad_volume_z" -c 2 -o gpurun_out/prof_fp_j python scripts/prof_step.py --what fp > gpurun_out/ncu_fp_j.log 2>&1; echo ncufull rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cone_fp_adjoint4z|unquad_z" -c 2 -o gpurun_out/prof_fpt_j python scripts/grad_bench.py --n 256 --views 180 --det 512 > gpurun_out/ncu_fpt_j.log 2>&1; echo ncufpt rc=$?
