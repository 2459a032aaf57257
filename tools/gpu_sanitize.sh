# compute-sanitizer over the GPU parity tests that exercise the hand-written mbarrier / TMA /
# tcgen05 / split-K pipelines: memcheck, racecheck, synccheck.
# Each tool runs only after the same pytest selection passed without it.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/sanitize
mkdir -p $O
SEL_OPS="tests/test_gpu_ops.py"
SEL_CNN="tests/test_gpu_unet.py -k conv_layer_vs_oracle_or_conv_pool_or_unet_forward_vs_reference_or_batched_vs_reference"
SEL_SOLVE="tests/test_gpu_solve.py -k n9"
run() {  # name, tool, selection...
  local name=$1 tool=$2; shift 2
  timeout 600 python -m pytest -m gpu -q -x "$@" > $O/plain_$name.log 2>&1 || { echo "$name: plain run failed"; tail -3 $O/plain_$name.log; return; }
  timeout 2400 compute-sanitizer --tool $tool --target-processes all --error-exitcode 99 --print-limit 20 \
    python -m pytest -m gpu -q -x -p no:cacheprovider "$@" > $O/${tool}_$name.log 2>&1
  echo "$name $tool rc=$? : $(grep -E 'ERROR SUMMARY|passed|failed' $O/${tool}_$name.log | tr '\n' ' ')"
}
for tool in memcheck synccheck racecheck; do
  run ops $tool $SEL_OPS
  run cnn $tool tests/test_gpu_unet.py -k "conv_layer_vs_oracle or conv_pool or unet_forward_vs_reference or batched_vs_reference"
  run solve $tool tests/test_gpu_solve.py -k "n9"
done
