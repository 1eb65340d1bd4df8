cd $GRAFT_REPO_ROOT
QRM_TRACE=1 python scripts/_scratch/dropin_quick.py 2>&1 | tail -14 | cut -c1-200
