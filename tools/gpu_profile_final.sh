cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/prof2
mkdir -p $O
timeout 500 python bench.py > $O/bench_full.log 2>&1
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-target > $O/bench_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-target > $O/ncu_launches.log 2>&1
timeout 300 python tools/cnn_one.py 33 1 2 > $O/plain_cnn33.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_split_reduce -s 2 -c 1 \
  -o $O/split_reduce_33 python tools/cnn_one.py 33 1 2 > $O/ncu_split_reduce.log 2>&1
timeout 600 python tools/step_breakdown.py --maxit 60 --out $O/breakdown_cfg2.json > $O/breakdown_cfg2.log 2>&1
ls -la $O
