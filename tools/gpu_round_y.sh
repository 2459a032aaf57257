cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | grep -E "^FAILED|passed|failed|Error|assert" | head -30 > gpurun_out/t_y.log
cat gpurun_out/t_y.log
timeout 600 python tools/step_breakdown.py --maxit 60 --out gpurun_out/breakdown_y.json > gpurun_out/breakdown_y.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --maxit 300 --no-cpu-baseline --no-target > gpurun_out/bench_y.log 2>&1
head -24 gpurun_out/breakdown_y.log; python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_y.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e'], d['iterations'], d['rel_residual'])
print({k:(round(v['ms']*1e3,1), round(v['tflops'],1)) for k,v in d['conv_layers'].items()})
PY
timeout 1500 python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline --no-target > gpurun_out/bench_cfg4_y.log 2>&1
timeout 2400 python bench.py --workload cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-target > gpurun_out/bench_cfg3_y.log 2>&1
tail -c 700 gpurun_out/bench_cfg4_y.log; tail -c 700 gpurun_out/bench_cfg3_y.log
