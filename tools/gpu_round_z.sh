cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | grep -E "^FAILED|passed|failed|Error|assert" | head -30 > gpurun_out/t_z.log
cat gpurun_out/t_z.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_z.log 2>&1; cat gpurun_out/smoke_z.log
timeout 600 python tools/step_breakdown.py --maxit 60 --out gpurun_out/breakdown_z.json > gpurun_out/breakdown_z.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_z.log 2>&1
head -24 gpurun_out/breakdown_z.log; python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_z.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e'], d['iterations'], d['rel_residual'], d.get('cpu_baseline'))
print({k:(round(v['ms']*1e3,1), round(v['tflops'],1)) for k,v in d['conv_layers'].items()})
print(json.dumps(d.get('target_128'))[:1500])
PY
