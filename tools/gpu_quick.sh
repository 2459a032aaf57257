cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_unet.py -q 2>&1 | tail -1
for cfg in "33 1" "129 1"; do set -- $cfg; echo "n=$1 $(timeout 300 python tools/cnn_breakdown.py --n $1 --nb $2 2>/dev/null | head -1)"; done
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --maxit 300 --no-cpu-baseline --no-target 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'])"; done
