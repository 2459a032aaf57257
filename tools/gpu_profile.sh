# Profiles for profiles/ (run under gpurun from the repo root, one GPU):
#  1. ncu launch list (gpu__time_duration) of the bench command (first 4000 launches)
#  2. ncu --set full of the dominant kernels at the bench size and the 128^3 target
#  3. warm in-graph breakdown and CNN breakdowns
# Each ncu pass runs only after the same command exited 0 without ncu.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/prof
mkdir -p $O
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-target > $O/bench_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-target > $O/ncu_launches.log 2>&1
run_full() {  # name, kernel regex, skip, command...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 300 "$@" > $O/plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c 1 \
    -o $O/$name "$@" > $O/ncu_$name.log 2>&1
}
run_full conv_dec1_33 conv3_tc_kernel 2 python tools/conv_one.py 33 64 32 0 3
run_full conv_enc2_33 conv3_tc_kernel 2 python tools/conv_one.py 33 32 64 1 3
run_full conv_dec1_129 conv3_tc_kernel 2 python tools/conv_one.py 129 64 32 0 3
run_full conv_enc2_129 conv3_tc_kernel 2 python tools/conv_one.py 129 32 64 1 3
run_full conv_enc3_65 conv3_tc_kernel 2 python tools/conv_one.py 65 64 128 1 3
run_full stencil_129x8 stencil_kernel 1 python tools/spmv_one.py 129 8 3 coupled
run_full stencil_33 stencil_kernel 1 python tools/spmv_one.py 33 1 3 coupled
run_full tconv_129 tconv_tc_kernel 3 python tools/cnn_one.py 129 1 2
timeout 600 python tools/step_breakdown.py --maxit 60 --out $O/breakdown_cfg2.json > $O/breakdown_cfg2.log 2>&1
for cfg in "129 1" "65 16" "33 1"; do set -- $cfg; timeout 300 python tools/cnn_breakdown.py --n $1 --nb $2 --out $O/cnn_$1_$2.json > /dev/null 2>&1; done
ls $O
