# Round-2 re-entry check: GPU suite (large-size oracle goldens still regenerating are deselected),
# smoke, the default (cfg4) bench line with its CPU baseline, then the ncu launch list of a short run.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/r2
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_large.py::test_cfg4_operators_vs_oracle \
  --deselect tests/test_gpu_large.py::test_cfg4_solve_head_vs_oracle --deselect tests/test_gpu_large.py::test_cfg3_batched_solve_head_vs_oracle \
  --deselect tests/test_gpu_large.py::test_cfg2_full_solve_outcome_vs_oracle --durations=15 > $O/tests_d.log 2>&1
tail -25 $O/tests_d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_d.log 2>&1
tail -2 $O/smoke_d.log
timeout 1500 python bench.py > $O/bench_d.log 2>&1
tail -c 6000 $O/bench_d.log
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref_d.log 2>&1
tail -c 1500 $O/bench_ref_d.log
timeout 900 python bench.py --steps 1 --warmup 1 --maxit 40 --no-cpu-baseline --no-target > $O/bench_short_d.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches_cfg4_d.csv \
  python bench.py --steps 1 --warmup 1 --maxit 40 --no-cpu-baseline --no-target > $O/ncu_launches_d.log 2>&1
tail -3 $O/ncu_launches_d.log
