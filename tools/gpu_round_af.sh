cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/spmv_one.py 129 8 3 coupled > gpurun_out/sp.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stencil|phase2" -s 4 -c 2 -o gpurun_out/prof_spmv_129x8 python tools/spmv_one.py 129 8 3 coupled > gpurun_out/ncu_af.log 2>&1
tail -2 gpurun_out/ncu_af.log
