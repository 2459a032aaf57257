# One-pass MGS Arnoldi: parity suite, A/B vs CGS2 (kernel and in-solve), FFMA2 microbenchmark.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/r2
mkdir -p $O
./tools/micro/ffma2_bench > $O/ffma2_e.log 2>&1; cat $O/ffma2_e.log
timeout 1800 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_large.py::test_cfg4_operators_vs_oracle \
  --deselect tests/test_gpu_large.py::test_cfg4_solve_head_vs_oracle --deselect tests/test_gpu_large.py::test_cfg3_batched_solve_head_vs_oracle \
  --deselect tests/test_gpu_large.py::test_cfg2_full_solve_outcome_vs_oracle > $O/tests_e.log 2>&1
tail -15 $O/tests_e.log
timeout 600 python tools/arnoldi_ab.py > $O/arnoldi_ab_e.log 2>&1; cat $O/arnoldi_ab_e.log
for orth in mgs cgs2; do
  MDP_ORTH=$orth timeout 900 python bench.py --workload cfg4 --maxit 200 --steps 2 --warmup 1 --no-cpu-baseline --no-target > $O/bench_cfg4_${orth}_e.log 2>&1
  python - <<PY
import json
d=json.loads(open("$O/bench_cfg4_${orth}_e.log").read().strip().splitlines()[-1])
print("cfg4 maxit200", "$orth", d["value"], d["ms_per_step"], d["rel_residual"], d["gpu_launches"])
PY
  MDP_ORTH=$orth timeout 900 python bench.py --workload cfg2 --steps 3 --warmup 2 --no-cpu-baseline --no-target > $O/bench_cfg2_${orth}_e.log 2>&1
  python - <<PY
import json
d=json.loads(open("$O/bench_cfg2_${orth}_e.log").read().strip().splitlines()[-1])
print("cfg2", "$orth", d["value"], d["ms_per_step"], d["rel_residual"], d["gpu_launches"])
PY
done
