cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "fused" > gpurun_out/r2/tests_c.log 2>&1
tail -3 gpurun_out/r2/tests_c.log
timeout 900 python tools/spmv_ab.py --cases cfg4,cfg2,129x8,65x16 --variants "V=3;V=4;V=4,NODES=16,ROWS=64;V=4,NODES=16,ROWS=64,LAST=1;V=4,NODES=8,ROWS=32;V=4,NODES=32,ROWS=128,LAST=1" > gpurun_out/r2/spmv_ab_c.log 2>&1
cat gpurun_out/r2/spmv_ab_c.log
