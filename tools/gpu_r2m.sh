# Staged tconv epilogue + capped ELL pull: parity tests, CNN breakdown A/B, SpMV A/B.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/r2
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_unet.py tests/test_gpu_large.py tests/test_gpu_ops.py tests/test_gpu_solve.py -m gpu -q -x -k "not cfg2_full" > $O/tests_m.log 2>&1
tail -n 5 $O/tests_m.log
for st in 0 1; do for n in 129 65 33; do
  MDP_TCONV_STAGED=$st timeout 300 python tools/cnn_breakdown.py --n $n > $O/cnn_breakdown_${n}_staged${st}.log 2>&1
  echo "staged=$st n=$n"; tail -n 2 $O/cnn_breakdown_${n}_staged${st}.log
done; done
timeout 600 python tools/spmv_ab.py --cases cfg4,cfg2,129x8,65x16 --variants "V=3" > $O/spmv_ab_m.log 2>&1; cat $O/spmv_ab_m.log
