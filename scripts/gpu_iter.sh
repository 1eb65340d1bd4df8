cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_hidden.py tests/test_cpp_dropin.py -x -q -m gpu 2>&1 | tail -3
for i in 1 2; do python scripts/bench_hidden.py 4096; done
