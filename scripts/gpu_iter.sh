cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_cpp_dropin.py -x -q -m gpu 2>&1 | tail -3
