# enc1a on tensor cores: CNN parity tests + forward breakdown A/B at 129^3 and 65^3.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_unet.py tests/test_gpu_large.py -m gpu -q -x -k "not cfg3 and not cfg2_full" > $O/tests_h.log 2>&1
tail -15 $O/tests_h.log
for tc in 0 1; do
  for n in 129 65; do
    MDP_ENC1A_TC=$tc timeout 300 python tools/cnn_breakdown.py --n $n > $O/cnn_breakdown_${n}_enc1atc${tc}.log 2>&1
    echo "enc1a_tc=$tc n=$n"; tail -2 $O/cnn_breakdown_${n}_enc1atc${tc}.log
  done
done
