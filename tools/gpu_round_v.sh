cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_ops.py -q 2>&1 | grep -E "^FAILED|passed|failed|Error|assert" | head -30 > gpurun_out/t_v.log
cat gpurun_out/t_v.log
timeout 900 python tools/stencil_sweep.py --z 0,8,16 > gpurun_out/sweep_v.log 2>&1
timeout 600 python tools/stencil_sweep.py --lib tools/ab/libst_ry4.so --z 0,8,16 > gpurun_out/sweep_v4.log 2>&1
cat gpurun_out/sweep_v*.log
