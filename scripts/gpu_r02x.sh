set -x
mkdir -p gpurun_out
timeout 900 python scripts/e2e_breakdown.py > gpurun_out/e2e_x.json 2> gpurun_out/e2e_x.err; echo e2e rc=$?
cat gpurun_out/e2e_x.json; tail -3 gpurun_out/e2e_x.err
