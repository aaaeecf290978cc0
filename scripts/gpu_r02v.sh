set -x
mkdir -p gpurun_out
timeout 900 python scripts/bench_variants.py --out gpurun_out/variants_v.json > gpurun_out/variants_v.log 2>&1; echo variants rc=$?
tail -12 gpurun_out/variants_v.log
timeout 1200 python scripts/bench_configs.py > gpurun_out/configs_v.json 2> gpurun_out/configs_v.err; echo configs rc=$?
tail -c 2000 gpurun_out/configs_v.json
