# Final-state check: whole GPU suite, smoke, the three bench lines and the reference arm.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/check
mkdir -p $O
(time timeout 3000 python -m pytest tests -m gpu -q -x) > $O/tests.log 2>&1; grep -E "passed|failed" $O/tests.log
timeout 600 python __graft_entry__.py smoke > $O/smoke.log 2>&1; tail -n 1 $O/smoke.log
(time timeout 1500 python bench.py) > $O/bench_cfg4.log 2>&1; tail -n 1 $O/bench_cfg4.log | cut -c1-200
(time timeout 900 python bench.py --impl reference) > $O/bench_cfg4_ref.log 2>&1; tail -n 1 $O/bench_cfg4_ref.log | cut -c1-200
(time timeout 1800 python bench.py --workload cfg3 --no-target) > $O/bench_cfg3.log 2>&1; tail -n 1 $O/bench_cfg3.log | cut -c1-200
(time timeout 900 python bench.py --workload cfg2 --no-target) > $O/bench_cfg2.log 2>&1; tail -n 1 $O/bench_cfg2.log | cut -c1-200
