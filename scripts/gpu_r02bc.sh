# Multi-rank bench paths run functionally on one GPU (gloo), after the round's FP launch changes.
set -x
mkdir -p gpurun_out
for f in zslab angle; do
TK_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --fdk $f --no-e2e --no-cpu-baseline > gpurun_out/bench_gloo2_${f}_bc.json 2> gpurun_out/bench_gloo2_${f}_bc.err; echo "$f rc=$?"
tail -c 400 gpurun_out/bench_gloo2_${f}_bc.json; tail -2 gpurun_out/bench_gloo2_${f}_bc.err
done
