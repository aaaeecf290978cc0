# Row-band FP pipeline, edge-inward schedule: device timing of the schedule, GPU pipeline tests, e2e breakdown.
set -x
mkdir -p gpurun_out
timeout 600 python scripts/fp_rows_probe.py > gpurun_out/fp_rows_aw.json 2>&1; echo probe rc=$?
tail -c 600 gpurun_out/fp_rows_aw.json
timeout 900 python -m pytest tests/test_gpu_pipeline.py -q -x > gpurun_out/pytest_pipe_aw.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_pipe_aw.log
for m in rows views; do
TK_FP_PIPE=$m timeout 600 python scripts/e2e_breakdown.py > gpurun_out/e2e_${m}_aw.json 2>/dev/null; echo "$m rc=$?"; cat gpurun_out/e2e_${m}_aw.json
done
timeout 600 python scripts/fp_pipe_timeline.py > gpurun_out/fp_pipe_tl_aw.json 2>/dev/null; echo tl rc=$?
