# Per-rank compute of the 2/4/8-GPU decompositions with the closing kernels.
set -x
mkdir -p gpurun_out
timeout 1500 python scripts/shard_model.py > gpurun_out/shard_model_be.json 2> gpurun_out/shard_model_be.err; echo shard rc=$?
cat gpurun_out/shard_model_be.json; tail -3 gpurun_out/shard_model_be.err
