set -x
mkdir -p gpurun_out
timeout 600 python scripts/e2e_breakdown.py > gpurun_out/e2e_param_ag.json 2> gpurun_out/e2e_param_ag.err; echo rc=$?
TK_UPLOAD=memcpy timeout 600 python scripts/e2e_breakdown.py > gpurun_out/e2e_memcpy_ag.json 2> gpurun_out/e2e_memcpy_ag.err; echo rc=$?
cat gpurun_out/e2e_param_ag.json gpurun_out/e2e_memcpy_ag.json; tail -3 gpurun_out/e2e_param_ag.err
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ag.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_ag.log
