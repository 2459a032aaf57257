cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python tools/arnoldi_ab.py tools/ab/libold.so > gpurun_out/arn_ab_r.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | grep -E "^FAILED|passed|failed|Error|assert" | head -30 > gpurun_out/t_r.log
timeout 1500 python tools/stencil_sweep.py > gpurun_out/sweep_r.log 2>&1
timeout 900 python tools/stencil_sweep.py --lib tools/ab/libst8.so --z 0,12,16,24 > gpurun_out/sweep_r8.log 2>&1
timeout 900 python tools/stencil_sweep.py --lib tools/ab/libst6.so --z 0,12,16,24 > gpurun_out/sweep_r6.log 2>&1
cat gpurun_out/arn_ab_r.log gpurun_out/t_r.log gpurun_out/sweep_r*.log
