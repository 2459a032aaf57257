# Round-2 final evidence: whole GPU suite, smoke, bench lines (cfg4 default + reference arm, cfg3, cfg2),
# launch list of the bench command, ncu --set full of the 129^3 CNN forward and the single-system cfg4 SpMV,
# cfg5 operator sweep, streamed SpMV timings.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/final
mkdir -p $O
(time timeout 3000 python -m pytest tests -m gpu -q -x) > $O/tests.log 2>&1; grep -E "passed|failed" $O/tests.log
timeout 600 python __graft_entry__.py smoke > $O/smoke.log 2>&1; tail -n 1 $O/smoke.log
(time timeout 1500 python bench.py) > $O/bench_cfg4.log 2>&1; tail -n 1 $O/bench_cfg4.log | cut -c1-200
(time timeout 900 python bench.py --impl reference) > $O/bench_cfg4_ref.log 2>&1; tail -n 1 $O/bench_cfg4_ref.log | cut -c1-200
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-target --maxit 150 > $O/bench_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches_bench_cfg4.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-target --maxit 150 > $O/ncu_launches.log 2>&1
python tools/launch_summary.py $O/launches_bench_cfg4.csv > $O/launches_bench_cfg4_summary.txt; head -n 8 $O/launches_bench_cfg4_summary.txt
(time timeout 1800 python bench.py --workload cfg3 --no-target) > $O/bench_cfg3.log 2>&1; tail -n 1 $O/bench_cfg3.log | cut -c1-200
(time timeout 900 python bench.py --workload cfg2 --no-target) > $O/bench_cfg2.log 2>&1; tail -n 1 $O/bench_cfg2.log | cut -c1-200
timeout 300 python tools/cnn_one.py 129 1 2 > $O/cnn_one_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"conv3_tc|tconv_tc|pack_input" -s 10 -c 10 -f -o $O/cnn_fwd_129 python tools/cnn_one.py 129 1 2 > $O/ncu_cnn_fwd.log 2>&1
timeout 300 python tools/spmv_one.py 0 1 3 coupled > $O/spmv_one_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil3_kernel|coupling_phase2" -s 2 -c 2 -f -o $O/spmv_cfg4_x1 python tools/spmv_one.py 0 1 3 coupled > $O/ncu_spmv.log 2>&1
timeout 900 python tools/stencil_stream.py --cases cfg4,129x8,65x16,cfg2,193x8,129x64 --variants base > $O/stencil_stream.log 2>&1
timeout 2400 python tools/bench_ops.py --out $O/ops_sweep_cfg5.json > $O/ops_sweep.log 2>&1; tail -n 2 $O/ops_sweep.log | cut -c1-300
for n in 129 65 33; do timeout 300 python tools/cnn_breakdown.py --n $n 2>/dev/null | tail -n 2; done > $O/cnn_breakdown.log; cat $O/cnn_breakdown.log
ls $O
