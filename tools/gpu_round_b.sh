cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python tools/diag_cfg1.py > gpurun_out/diag_cfg1.log 2>&1
timeout 300 python -m pytest tests/test_gpu_ops.py -q -k batched_engine 2>&1 | tail -5 >> gpurun_out/diag_cfg1.log
cat gpurun_out/diag_cfg1.log
