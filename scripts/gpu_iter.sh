cd $GRAFT_REPO_ROOT
QRM_DEBUG_STAGES=1 timeout 300 python scripts/dbg_corr.py 2>&1 | grep "qrm stages" | head -12
