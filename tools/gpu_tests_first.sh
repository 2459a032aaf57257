cd $GRAFT_REPO_ROOT
nvidia-smi -L
export PYTHONDONTWRITEBYTECODE=1
timeout 400 python -m pytest tests/test_gpu_ops.py -q -x 2>&1 | tail -30 > gpurun_out/t_ops.log
timeout 300 python -m pytest tests/test_gpu_unet.py -q -k "path1 or (test_conv_layer_vs_oracle and -1-)" 2>&1 | tail -30 > gpurun_out/t_unet1.log
timeout 120 python -m pytest tests/test_gpu_unet.py -q -x -k "test_conv_layer_vs_oracle and 0-32-64-8" 2>&1 | tail -30 > gpurun_out/t_unet0.log
cat gpurun_out/t_ops.log gpurun_out/t_unet1.log gpurun_out/t_unet0.log
