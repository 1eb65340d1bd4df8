cd $GRAFT_REPO_ROOT
for f in 2 4 0; do echo "== flags $f"; QRM_EXP_FLAGS=$f KS=0 python scripts/sweep_corr.py 2>&1 | grep -E "batch': (4096|16384|65536)"; done
for g in 64 32; do echo "== flags 2 + L2 fetch $g"; QRM_L2_FETCH=$g QRM_EXP_FLAGS=2 KS=0 python scripts/sweep_corr.py 2>&1 | grep -E "batch': (4096|16384|65536)"; done
echo "== flags 4 + L2 fetch 64"; QRM_L2_FETCH=64 QRM_EXP_FLAGS=4 KS=0 python scripts/sweep_corr.py 2>&1 | grep -E "batch': (4096|16384|65536)"
