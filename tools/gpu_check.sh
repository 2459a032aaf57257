# Round-end style check on a GPU box (run under gpurun from the repo root):
#   GPU test suite, smoke(), the default bench line and the reference arm.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/check_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/check_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/check_bench_ref.log 2>&1
tail -3 gpurun_out/check_tests.log; cat gpurun_out/check_smoke.log; tail -c 400 gpurun_out/check_bench.log; tail -c 300 gpurun_out/check_bench_ref.log
if [ "${WITH_CFG34:-0}" = "1" ]; then
  timeout 1500 python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline --no-target > gpurun_out/check_bench_cfg4.log 2>&1
  timeout 2400 python bench.py --workload cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-target > gpurun_out/check_bench_cfg3.log 2>&1
  tail -c 300 gpurun_out/check_bench_cfg4.log; tail -c 300 gpurun_out/check_bench_cfg3.log
fi
