# Whole GPU suite on the current build, default bench, ncu of the single-system cfg4 coupled SpMV.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/r2
mkdir -p $O
(time timeout 3000 python -m pytest tests -m gpu -q -x --durations=10 --deselect tests/test_gpu_large.py::test_cfg2_full_solve_outcome_vs_oracle) > $O/tests_l.log 2>&1
tail -n 18 $O/tests_l.log
timeout 300 python tools/spmv_one.py 0 1 3 coupled > $O/spmv_one_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil3_kernel|coupling_phase2" -s 2 -c 2 -f -o $O/spmv_cfg4_x1 python tools/spmv_one.py 0 1 3 coupled > $O/ncu_spmv.log 2>&1
tail -n 2 $O/ncu_spmv.log
(time timeout 1500 python bench.py) > $O/bench_default_l.log 2>&1; tail -n 1 $O/bench_default_l.log | cut -c1-600
