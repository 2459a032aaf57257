cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | grep -E "^FAILED|passed|failed|Error|assert" | head -30 > gpurun_out/t_ah.log
cat gpurun_out/t_ah.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for pdl in 1 0; do
MDP_PDL=$pdl timeout 600 python tools/step_breakdown.py --maxit 60 > gpurun_out/breakdown_ah_$pdl.log 2>&1
MDP_PDL=$pdl timeout 600 python bench.py --steps 3 --warmup 3 --maxit 300 --no-cpu-baseline --no-target > gpurun_out/bench_ah_$pdl.log 2>&1
echo "PDL=$pdl"; sed -n 3p gpurun_out/breakdown_ah_$pdl.log | cut -c1-300
python -c "
import json; d=json.loads(open('gpurun_out/bench_ah_$pdl.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'])"
done
