# Mirror-pair forward projector: parity, then cfg4 timing of each launch configuration vs the general kernel.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "Mirror or Golden or Oracle" > gpurun_out/pytest_b.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_b.log
timeout 900 python scripts/fp_sweep.py --op fp --reps 3 --configs "TK_FP_MIRROR=0;TK_FP_MIRROR=1,TK_FPM_CFG=4x3;TK_FPM_CFG=8x1;TK_FPM_CFG=8x2" > gpurun_out/fpm_sweep_b.json 2>&1; echo sweep rc=$?
cat gpurun_out/fpm_sweep_b.json
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "Cfg3 or Cfg4" > gpurun_out/pytest_cfg_b.log 2>&1; echo cfg rc=$?
tail -3 gpurun_out/pytest_cfg_b.log
