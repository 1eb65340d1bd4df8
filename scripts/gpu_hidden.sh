cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_hidden.py -x -q -m gpu -s > gpurun_out/hidden_test.log 2>&1; echo "rc=$?" >> gpurun_out/hidden_test.log
tail -4 gpurun_out/hidden_test.log
timeout 120 python scripts/bench_hidden.py 4096 2>&1 | tail -1
timeout 120 python scripts/bench_hidden.py 1024 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:conv64 -s 10 -c 1 -o gpurun_out/conv64c python scripts/bench_hidden.py 512 > gpurun_out/ncu_conv.log 2>&1; tail -1 gpurun_out/ncu_conv.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/bench_hidden.py 512 2>/dev/null | grep -E "conv|hidden" | tail -12 > gpurun_out/hidden_launches.csv
