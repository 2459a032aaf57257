cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_unet.py tests/test_gpu_solve.py -q -x -k "not cfg1" 2>&1 | tail -30 > gpurun_out/t_d.log
timeout 1200 python bench.py --steps 2 --warmup 1 --maxit 300 --no-cpu-baseline > gpurun_out/bench_d.log 2>&1
python tools/profile_step.py --maxit 4 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_d.csv python tools/profile_step.py --maxit 4 --reps 2 > gpurun_out/ncu_d.log 2>&1
tail -n 5 gpurun_out/t_d.log; head -c 400 gpurun_out/bench_d.log
