cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | grep -E "^FAILED|passed|failed|Error|assert" | head -30 > gpurun_out/t_q.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_q.log 2>&1
timeout 600 python tools/arnoldi_ab.py tools/ab/libold.so > gpurun_out/arn_ab_q.log 2>&1
timeout 600 python tools/step_breakdown.py --maxit 60 --out gpurun_out/breakdown_q.json > gpurun_out/breakdown_q.log 2>&1
timeout 300 python tools/cnn_one.py 33 1 3 > gpurun_out/cnn_plain_q.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tconv|enc1a|pack_input|split_reduce" -s 6 -c 6 -o gpurun_out/prof_cnn_small_33 python tools/cnn_one.py 33 1 3 > gpurun_out/ncu_cnn33.log 2>&1
cat gpurun_out/t_q.log gpurun_out/smoke_q.log gpurun_out/arn_ab_q.log; head -30 gpurun_out/breakdown_q.log
