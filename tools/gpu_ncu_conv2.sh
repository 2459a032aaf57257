cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 120 python tools/conv_one.py 129 64 32 0 3 > gpurun_out/conv_one_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3_tc_kernel -s 2 -c 1 -o gpurun_out/prof_dec1_129b python tools/conv_one.py 129 64 32 0 3 > gpurun_out/ncu_conv2.log 2>&1
tail -2 gpurun_out/ncu_conv2.log
