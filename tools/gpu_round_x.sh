cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python tools/stencil_sweep.py --z 0,16 > gpurun_out/sweep_x2.log 2>&1
timeout 600 python tools/stencil_sweep.py --lib tools/ab/libst_pf3.so --z 0,16,32 > gpurun_out/sweep_x3.log 2>&1
timeout 600 python tools/stencil_sweep.py --lib tools/ab/libst_pf4.so --z 0,16,32 > gpurun_out/sweep_x4.log 2>&1
cat gpurun_out/sweep_x*.log
