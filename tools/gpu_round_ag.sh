cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
for t in u2 u6 r4 r4u2 r3; do echo "== $t"; timeout 600 python tools/stencil_sweep.py --lib tools/ab/libst_$t.so --z 0,16 2>&1; done
echo "== cur"; timeout 300 python tools/stencil_sweep.py --z 0 2>&1
