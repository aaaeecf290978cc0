set -x
mkdir -p gpurun_out
timeout 900 python scripts/fp_band_probe.py > gpurun_out/fp_band_d.log 2>&1; echo probe rc=$?
cat gpurun_out/fp_band_d.log
