cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_unet.py -q 2>&1 | tail -40 > gpurun_out/t_a.log
timeout 900 python -m pytest tests/test_gpu_solve.py -q 2>&1 | tail -40 > gpurun_out/t_solve.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py --steps 1 --warmup 1 --maxit 300 > gpurun_out/bench_a.log 2>&1
tail -5 gpurun_out/t_a.log gpurun_out/t_solve.log gpurun_out/smoke.log gpurun_out/bench_a.log
