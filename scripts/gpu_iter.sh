cd $GRAFT_REPO_ROOT
timeout 120 python -m pytest tests/test_hidden.py -x -q -m gpu > gpurun_out/t.log 2>&1; echo "tests rc=$?" >> gpurun_out/t.log; tail -2 gpurun_out/t.log
QRM_CONV_PAIR=0 timeout 120 python -m pytest tests/test_hidden.py -x -q -m gpu 2>&1 | tail -1
for pr in 1 0 1 0; do QRM_CONV_PAIR=$pr timeout 120 python scripts/bench_hidden.py 4096 2>&1 | tail -1; done
