# Round-2 evidence: whole GPU suite, default bench + reference arm, launch list, cfg3/cfg2 lines, CNN forward ncu.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/r2o
mkdir -p $O
(time timeout 3000 python -m pytest tests -m gpu -q -x) > $O/tests.log 2>&1; tail -n 4 $O/tests.log
timeout 600 python __graft_entry__.py smoke > $O/smoke.log 2>&1; tail -n 1 $O/smoke.log
(time timeout 1500 python bench.py) > $O/bench_cfg4.log 2>&1; tail -n 1 $O/bench_cfg4.log | cut -c1-300
(time timeout 900 python bench.py --impl reference) > $O/bench_cfg4_ref.log 2>&1; tail -n 1 $O/bench_cfg4_ref.log | cut -c1-200
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-target --maxit 150 > $O/bench_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches_bench_cfg4.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-target --maxit 150 > $O/ncu_launches.log 2>&1
python tools/launch_summary.py $O/launches_bench_cfg4.csv > $O/launches_bench_cfg4_summary.txt; head -n 12 $O/launches_bench_cfg4_summary.txt
(time timeout 1800 python bench.py --workload cfg3 --no-target) > $O/bench_cfg3.log 2>&1; tail -n 1 $O/bench_cfg3.log | cut -c1-300
(time timeout 900 python bench.py --workload cfg2 --no-target) > $O/bench_cfg2.log 2>&1; tail -n 1 $O/bench_cfg2.log | cut -c1-300
timeout 300 python tools/cnn_one.py 129 1 2 > $O/cnn_one_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"conv3_tc|tconv_tc|pack_input" -s 10 -c 10 -f -o $O/cnn_fwd_129 python tools/cnn_one.py 129 1 2 > $O/ncu_cnn_fwd.log 2>&1
tail -n 1 $O/ncu_cnn_fwd.log
