cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python tools/bench_ops.py --sizes 33,65,129,193 --batches 1,8,64 --out gpurun_out/ops_sweep.json > gpurun_out/ops_sweep.log 2>&1
tail -c 3000 gpurun_out/ops_sweep.log
