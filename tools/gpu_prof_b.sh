cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/profile_step.py --maxit 4 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_j.csv python tools/profile_step.py --maxit 4 --reps 2 > gpurun_out/ncu_j.log 2>&1
tail -1 gpurun_out/ncu_j.log
