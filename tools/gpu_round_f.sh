cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_unet.py tests/test_gpu_ops.py -q -x 2>&1 | tail -3 > gpurun_out/t_f.log
timeout 600 python tools/conv_bench.py 33 65 129 > gpurun_out/conv_f.log 2>&1
cat gpurun_out/t_f.log gpurun_out/conv_f.log
