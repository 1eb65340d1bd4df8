cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_hidden.py -x -q -m gpu -s > gpurun_out/hidden_test.log 2>&1; echo "rc=$?" >> gpurun_out/hidden_test.log
tail -15 gpurun_out/hidden_test.log
timeout 120 python scripts/bench_hidden.py 1024 2>&1 | tail -3
timeout 120 python scripts/bench_hidden.py 4096 2>&1 | tail -3
