cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
for z in 0 1 2 3 4 6; do
  if [ $z = 0 ]; then unset MDP_STENCIL_ZCHUNK; else export MDP_STENCIL_ZCHUNK=$z; fi
  echo "zchunk=$z $(timeout 600 python bench.py --steps 3 --warmup 3 --maxit 300 --no-cpu-baseline --no-target 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],3), round(d["ms_per_step"],1))')"
done
