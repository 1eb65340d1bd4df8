cd $GRAFT_REPO_ROOT
for pr in 1 0; do echo "pair=$pr"; QRM_CONV_PAIR=$pr ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:conv64 -s 3 -c 1 python scripts/bench_hidden.py 1024 2>/dev/null | grep -E "duration|tensor"; done
QRM_CONV_PAIR=1 timeout 300 python -m pytest tests/test_hidden.py -x -q -m gpu 2>&1 | tail -1
