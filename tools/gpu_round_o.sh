cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | grep -E "^FAILED|passed|failed|Error" | head -20 > gpurun_out/t_o.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_o.log 2>&1
timeout 600 python tools/step_breakdown.py --maxit 60 --out gpurun_out/breakdown_o.json > gpurun_out/breakdown_o.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_o.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_o.log 2>&1
cat gpurun_out/t_o.log gpurun_out/smoke_o.log; head -40 gpurun_out/breakdown_o.log; tail -c 600 gpurun_out/bench_o.log; tail -c 400 gpurun_out/bench_ref_o.log
