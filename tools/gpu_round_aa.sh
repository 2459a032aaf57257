cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
for cfg in "129 1" "65 16" "33 1"; do set -- $cfg; timeout 300 python tools/cnn_breakdown.py --n $1 --nb $2 --out gpurun_out/cnnbd_$1_$2.json > gpurun_out/cnnbd_$1_$2.log 2>&1; done
timeout 300 python tools/conv_one.py 32 128 128 0 3 > gpurun_out/c1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3_tc_kernel -s 2 -c 1 -o gpurun_out/prof_conv_bott_32 python tools/conv_one.py 32 128 128 0 3 > gpurun_out/ncu_aa1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3_tc_kernel -s 2 -c 1 -o gpurun_out/prof_conv_enc2_129 python tools/conv_one.py 129 32 64 1 3 > gpurun_out/ncu_aa2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3_tc_kernel -s 2 -c 1 -o gpurun_out/prof_conv_dec1f_129 python tools/conv_one.py 129 64 32 0 3 > gpurun_out/ncu_aa3.log 2>&1
cat gpurun_out/cnnbd_*.log
