mkdir -p gpurun_out
(timeout 60 ./scripts/tmatest/tma_cccl; for m in 32 36 40 33; do timeout 60 ./scripts/tmatest/tma_min $m; done) > gpurun_out/tma_dbg2.log 2>&1
cat gpurun_out/tma_dbg2.log
