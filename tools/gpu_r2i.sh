# ncu --set full of one whole CNN forward at 129^3 (10 launches, second forward)
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
O=gpurun_out/r2
mkdir -p $O
timeout 300 python tools/cnn_one.py 129 1 2 > $O/cnn_one_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -s 10 -c 10 -f -o $O/cnn_fwd_129 python tools/cnn_one.py 129 1 2 > $O/ncu_cnn_fwd.log 2>&1
tail -3 $O/ncu_cnn_fwd.log; ls -la $O/*.ncu-rep
