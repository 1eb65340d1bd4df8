cd $GRAFT_REPO_ROOT
for d in 0 32 16; do echo "pair dbg=$d"; QRM_HIDDEN_DBG=$d ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:conv64 -s 3 -c 1 python scripts/bench_hidden.py 1024 2>/dev/null | grep -E "duration|tensor"; done
