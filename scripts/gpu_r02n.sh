# Full GPU suite + smoke after the 2D centre-relative change; cfg5 gradient / transpose timings; ncu of A^T.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_n.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_n.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_n.log 2>&1; echo smoke rc=$?
cat gpurun_out/smoke_n.log
timeout 600 python scripts/grad_bench.py > gpurun_out/grad_n.json 2> gpurun_out/grad_n.err; echo grad rc=$?
cat gpurun_out/grad_n.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"cone_fp_adjoint4z_kernel" -c 1 -o gpurun_out/prof_fpt_n python scripts/prof_adjoint.py > gpurun_out/ncu_fpt_n.log 2>&1; echo ncu rc=$?
