cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python tools/conv_variants.py > gpurun_out/conv_var.log 2>&1
cat gpurun_out/conv_var.log
