cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests/test_gpu_unet.py -q -x 2>&1 | grep -E "^FAILED|passed|failed|Error|assert" | head -30 > gpurun_out/t_ad.log
cat gpurun_out/t_ad.log
for cfg in "129 1" "65 16" "33 1"; do set -- $cfg; timeout 300 python tools/cnn_breakdown.py --n $1 --nb $2 --out gpurun_out/cnnbd_$1_$2.json > gpurun_out/cnnbd_$1_$2.log 2>&1; done
timeout 600 python bench.py --steps 3 --warmup 3 --maxit 300 --no-cpu-baseline > gpurun_out/bench_ad.log 2>&1
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_ad.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e'])
print({k:(round(v['ms']*1e3,1), round(v['tflops'],1)) for k,v in d['conv_layers'].items()})
print(json.dumps(d.get('target_128'))[:1500])
PY
