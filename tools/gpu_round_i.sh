cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_unet.py tests/test_gpu_ops.py tests/test_gpu_solve.py -q -k "not cfg1" 2>&1 | grep -E "^FAILED|passed|failed" | head -20 > gpurun_out/t_i.log
timeout 300 python tools/conv_bench.py 33 65 129 > gpurun_out/conv_i.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_i.log 2>&1
timeout 1200 python bench.py --steps 2 --warmup 1 --maxit 300 --no-cpu-baseline > gpurun_out/bench_i.log 2>&1
cat gpurun_out/t_i.log gpurun_out/conv_i.log gpurun_out/smoke_i.log; head -c 400 gpurun_out/bench_i.log
