cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_unet.py tests/test_gpu_solve.py -q -x -k "not cfg1" 2>&1 | tail -5 > gpurun_out/t_e.log
timeout 600 python tools/conv_bench.py 33 65 129 > gpurun_out/conv_e.log 2>&1
timeout 1200 python bench.py --steps 2 --warmup 1 --maxit 300 --no-cpu-baseline > gpurun_out/bench_e.log 2>&1
cat gpurun_out/t_e.log gpurun_out/conv_e.log; head -c 300 gpurun_out/bench_e.log
