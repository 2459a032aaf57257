cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_unet.py tests/test_gpu_solve.py -q 2>&1 | grep -E "^FAILED|passed|failed|Error" | head -20 > gpurun_out/t_l.log
timeout 900 python tools/bench_ops.py --sizes 33,65,129,193 --batches 1,8 --out gpurun_out/ops_sweep_l.json > gpurun_out/ops_l.log 2>&1
timeout 1200 python bench.py --steps 2 --warmup 1 --maxit 300 --no-cpu-baseline > gpurun_out/bench_l.log 2>&1
cat gpurun_out/t_l.log; head -c 300 gpurun_out/bench_l.log
