set -x
mkdir -p gpurun_out
timeout 1500 python scripts/shard_model.py > gpurun_out/shard_model_ab.json 2> gpurun_out/shard_model_ab.err; echo shard rc=$?
cat gpurun_out/shard_model_ab.json; tail -3 gpurun_out/shard_model_ab.err
