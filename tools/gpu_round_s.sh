cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^FAILED|passed|failed|Error|assert" | head -30 > gpurun_out/t_s.log
timeout 900 python tools/arnoldi_ab.py tools/ab/libold.so tools/ab/libk_*.so > gpurun_out/arn_ab_s.log 2>&1
timeout 600 python tools/step_breakdown.py --maxit 60 --out gpurun_out/breakdown_s.json > gpurun_out/breakdown_s.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --maxit 300 --no-cpu-baseline > gpurun_out/bench_s.log 2>&1
cat gpurun_out/t_s.log gpurun_out/arn_ab_s.log; head -24 gpurun_out/breakdown_s.log; tail -c 1500 gpurun_out/bench_s.log
