cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_unet.py tests/test_gpu_solve.py -q 2>&1 | grep -E "^FAILED|passed|failed|Error|assert" | head -20
for cfg in "129 1" "65 16" "33 1"; do set -- $cfg; timeout 300 python tools/cnn_breakdown.py --n $1 --nb $2 > gpurun_out/cnnbd_$1_$2.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/cnnbd_$1_$2.log').read()); print('$1x$2', round(d['forward_ms'],3), round(d['tflops'],1), {k[:24]:v for k,v in list(d['kernels_us_per_forward'].items())[:5]})"; done
