cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/spmv_one.py 129 4 3 > gpurun_out/spmv_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 2 -c 1 -o gpurun_out/prof_stencil python tools/spmv_one.py 129 4 3 > gpurun_out/ncu_st.log 2>&1
tail -2 gpurun_out/ncu_st.log
