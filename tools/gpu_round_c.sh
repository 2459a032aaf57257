cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_unet.py tests/test_gpu_solve.py -q -x -k "not cfg1" 2>&1 | tail -30 > gpurun_out/t_c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_c.log 2>&1
timeout 1200 python bench.py --steps 2 --warmup 1 --maxit 300 --no-cpu-baseline > gpurun_out/bench_c.log 2>&1
tail -n 5 gpurun_out/t_c.log gpurun_out/smoke_c.log; tail -c 1500 gpurun_out/bench_c.log
