cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests/test_gpu_unet.py -q -x 2>&1 | tail -3 > gpurun_out/t_h.log
timeout 300 python tools/conv_bench.py 33 65 129 > gpurun_out/conv_h.log 2>&1
cat gpurun_out/t_h.log gpurun_out/conv_h.log
