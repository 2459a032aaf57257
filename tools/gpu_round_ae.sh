cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
for ad in 4 6 8; do timeout 600 python tools/stencil_sweep.py --lib tools/ab/libst_async$ad.so --z 0,16,32 > gpurun_out/sweep_async$ad.log 2>&1; done
timeout 300 python tools/stencil_sweep.py --z 0 > gpurun_out/sweep_cur.log 2>&1
for f in gpurun_out/sweep_async*.log gpurun_out/sweep_cur.log; do echo $f; cat $f; done
