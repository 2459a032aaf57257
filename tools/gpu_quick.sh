cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_solve.py -q 2>&1 | tail -2
timeout 600 python tools/step_breakdown.py --maxit 60 2>/dev/null | sed -n 2,14p
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --maxit 300 --no-cpu-baseline --no-target 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'])"; done
