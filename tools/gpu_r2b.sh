# Round-2 probe: stencil/coupled SpMV at single systems (cold L2) and the warm kernel
# breakdown of one CNN forward at 129^3 / 33^3.
cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONDONTWRITEBYTECODE=1
mkdir -p gpurun_out/r2
timeout 600 python tools/stencil_ab.py --versions 3 --cases 33x1,65x1,129x1,129x8,193x1 > gpurun_out/r2/stencil_ab_b.log 2>&1
cat gpurun_out/r2/stencil_ab_b.log
timeout 600 python tools/cnn_breakdown.py --n 129 --out gpurun_out/r2/cnn129_breakdown.json > gpurun_out/r2/cnn129_b.log 2>&1
cat gpurun_out/r2/cnn129_b.log
timeout 600 python tools/cnn_breakdown.py --n 33 --out gpurun_out/r2/cnn33_breakdown.json > gpurun_out/r2/cnn33_b.log 2>&1
cat gpurun_out/r2/cnn33_b.log
