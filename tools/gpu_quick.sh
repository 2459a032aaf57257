cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
for pdl in 0 1; do for lib in "" tools/ab/libtc_old.so; do for cfg in "129 1" "65 16" "33 1"; do set -- $cfg
echo "pdl=$pdl lib=${lib:-cur} n=$1 nb=$2 $(MDP_PDL=$pdl timeout 300 python tools/cnn_breakdown.py --n $1 --nb $2 ${lib:+--lib $lib} 2>/dev/null | head -1)"
done; done; done
