cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
python tools/profile_step.py --maxit 4 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/profile_step.py --maxit 4 --reps 2 > gpurun_out/ncu_a.log 2>&1
tail -3 gpurun_out/ncu_a.log; wc -l gpurun_out/launches_cfg2.csv
