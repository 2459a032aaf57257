cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_solve.py -q 2>&1 | grep -E "^FAILED|passed|failed|Error" | head -20 > gpurun_out/t_m.log
timeout 900 python tools/bench_ops.py --sizes 65,129,193 --batches 1,8 --out gpurun_out/ops_sweep_m.json > gpurun_out/ops_m.log 2>&1
cat gpurun_out/t_m.log
