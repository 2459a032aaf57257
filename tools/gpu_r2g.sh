# Re-entry check: whole GPU parity suite, smoke, default bench line (cfg4) + reference arm.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/r2
mkdir -p $O
(time timeout 2400 python -m pytest tests -m gpu -q -x --durations=15) > $O/tests_g.log 2>&1
tail -30 $O/tests_g.log
timeout 600 python __graft_entry__.py smoke > $O/smoke_g.log 2>&1; tail -3 $O/smoke_g.log
(time timeout 1500 python bench.py) > $O/bench_default_g.log 2>&1; tail -5 $O/bench_default_g.log
(time timeout 900 python bench.py --impl reference) > $O/bench_ref_g.log 2>&1; tail -5 $O/bench_ref_g.log
