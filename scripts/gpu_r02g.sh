# ncu: full capture (with source) of the general forward kernel at cfg4; DRAM / hit-rate metrics of the
# segmented and mirror variants.
set -x
mkdir -p gpurun_out
export TK_FP_MIRROR=0
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"cone_fp_kernel" -c 1 -o gpurun_out/prof_fp_g python scripts/prof_step.py --what fp > gpurun_out/ncu_fp_g.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_fp_g.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
for cfg in "TK_FP_MIRROR=0 TK_FP_SEG=2" "TK_FP_MIRROR=1 TK_FP_SEG=1" "TK_FP_MIRROR=1 TK_FP_SEG=2"; do
  env $cfg timeout 900 ncu --metrics $M --clock-control none -k regex:"cone_fp" --csv python scripts/prof_step.py --what fp > "gpurun_out/ncu_m_g_${cfg// /_}.csv" 2>&1; echo m rc=$?
done
