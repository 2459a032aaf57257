cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/spmv_one.py 129 8 3 > gpurun_out/spmv_plain_w.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_bulk -s 2 -c 1 -o gpurun_out/prof_stencil_bulk_w python tools/spmv_one.py 129 8 3 > gpurun_out/ncu_w.log 2>&1
tail -3 gpurun_out/ncu_w.log
