# ncu full capture of the mirror-pair forward projector at cfg4 (720 views).
set -x
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cone_fp_mirror_kernel" -c 1 -o gpurun_out/prof_fpm_c python scripts/prof_step.py --what fp > gpurun_out/ncu_fpm_c.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_fpm_c.log
