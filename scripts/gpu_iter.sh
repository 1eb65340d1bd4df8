cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:conv0 -s 2 -c 1 python scripts/bench_hidden.py 1024 2>/dev/null | grep -E "duration|write"
timeout 300 python -m pytest tests/test_hidden.py -x -q -m gpu 2>&1 | tail -1
