# Wide-basis Arnoldi kernel + Jacobi operands through the stage ring: parity suite, A/Bs, bench lines.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/r2
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_large.py::test_cfg4_operators_vs_oracle \
  --deselect tests/test_gpu_large.py::test_cfg4_solve_head_vs_oracle --deselect tests/test_gpu_large.py::test_cfg3_batched_solve_head_vs_oracle \
  --deselect tests/test_gpu_large.py::test_cfg2_full_solve_outcome_vs_oracle > $O/tests_f.log 2>&1
tail -15 $O/tests_f.log
timeout 600 python tools/arnoldi_ab.py > $O/arnoldi_ab_f.log 2>&1; cat $O/arnoldi_ab_f.log
timeout 600 python tools/spmv_ab.py --cases cfg4,cfg2,129x8,65x16 --variants "V=3" > $O/spmv_ab_f.log 2>&1; cat $O/spmv_ab_f.log
for wl in cfg4 cfg3; do
  timeout 900 python bench.py --workload $wl --maxit 200 --steps 2 --warmup 1 --no-cpu-baseline --no-target > $O/bench_${wl}_f.log 2>&1
  python - <<PY
import json
d=json.loads(open("$O/bench_${wl}_f.log").read().strip().splitlines()[-1])
print("$wl maxit200", d["value"], d["ms_per_step"], d["rel_residual"][:2], d["gpu_launches"], d["applies_per_s"])
PY
done
timeout 900 python bench.py --workload cfg2 --steps 3 --warmup 2 --no-cpu-baseline --no-target > $O/bench_cfg2_f.log 2>&1
python - <<PY
import json
d=json.loads(open("$O/bench_cfg2_f.log").read().strip().splitlines()[-1])
print("cfg2", d["value"], d["ms_per_step"], d["rel_residual"], d["gpu_launches"], d["applies_per_s"])
PY
