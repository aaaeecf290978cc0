set -x
mkdir -p gpurun_out
timeout 900 python scripts/e2e_parts.py > gpurun_out/e2e_parts_z.log 2>&1; echo parts rc=$?
cat gpurun_out/e2e_parts_z.log
