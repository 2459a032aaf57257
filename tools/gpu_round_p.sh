cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -q -x -k "not cfg1_reference_semantics" 2>&1 | grep -E "^FAILED|passed|failed|Error" | head -20 > gpurun_out/t_p.log
timeout 600 python -m pytest tests/test_gpu_solve.py -q -k "cfg1_reference_semantics" 2>&1 | tail -40 > gpurun_out/t_p_cfg1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_p.log 2>&1
timeout 600 python tools/step_breakdown.py --maxit 60 --out gpurun_out/breakdown_p.json > gpurun_out/breakdown_p.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_p.log 2>&1
timeout 900 python tools/bench_ops.py --sizes 33,65,129,193 --batches 1,8 --out gpurun_out/ops_sweep_p.json > gpurun_out/ops_p.log 2>&1
# launch list of the bench command (first 4000 launches of the warm-up solves)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_bench_p.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-target > gpurun_out/ncu_launch_p.log 2>&1
# full captures of the top kernels
timeout 300 python tools/conv_one.py 33 64 32 0 3 > gpurun_out/conv_plain_p.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3_tc_kernel -s 2 -c 1 -o gpurun_out/prof_conv_dec1_33 python tools/conv_one.py 33 64 32 0 3 > gpurun_out/ncu_c33.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3_tc_kernel -s 2 -c 1 -o gpurun_out/prof_conv_dec1_129 python tools/conv_one.py 129 64 32 0 3 > gpurun_out/ncu_c129.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv3_tc_kernel -s 2 -c 1 -o gpurun_out/prof_conv_enc3_65 python tools/conv_one.py 65 64 128 1 3 > gpurun_out/ncu_c65.log 2>&1
timeout 300 python tools/spmv_one.py 129 1 3 > gpurun_out/spmv_plain_p.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 2 -c 1 -o gpurun_out/prof_stencil_129 python tools/spmv_one.py 129 1 3 > gpurun_out/ncu_st_p.log 2>&1
cat gpurun_out/t_p.log gpurun_out/smoke_p.log; head -30 gpurun_out/breakdown_p.log; tail -c 800 gpurun_out/bench_p.log
