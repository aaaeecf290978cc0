mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python scripts/e2e_breakdown.py > gpurun_out/e2e_s1_aj.json 2>/dev/null; cat gpurun_out/e2e_s1_aj.json
TK_PIPE_STREAMS=2 timeout 600 python scripts/e2e_breakdown.py > gpurun_out/e2e_s2_aj.json 2>/dev/null; cat gpurun_out/e2e_s2_aj.json
done
