cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_unet.py -q 2>&1 | grep -E "^FAILED|passed|failed|Error|assert" | head -30 > gpurun_out/t_ac.log
cat gpurun_out/t_ac.log
for cfg in "129 1" "65 16" "33 1"; do set -- $cfg; timeout 300 python tools/cnn_breakdown.py --n $1 --nb $2 --out gpurun_out/cnnbd_$1_$2.json > gpurun_out/cnnbd_$1_$2.log 2>&1; done
timeout 300 python tools/cnn_one.py 129 1 2 > gpurun_out/cnn129.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tconv_tc|enc1a" -s 3 -c 3 -o gpurun_out/prof_tconv_129 python tools/cnn_one.py 129 1 2 > gpurun_out/ncu_ac.log 2>&1
tail -2 gpurun_out/ncu_ac.log
