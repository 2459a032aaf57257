# Round-2 first check: GPU suite (without the large-size goldens still being generated),
# smoke, and a short cfg4 bench line.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_large.py > gpurun_out/r2/tests_a.log 2>&1
tail -5 gpurun_out/r2/tests_a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke_a.log 2>&1
tail -2 gpurun_out/r2/smoke_a.log
timeout 1200 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2/bench_a.log 2>&1
tail -c 3000 gpurun_out/r2/bench_a.log
