cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_rs.py -x -q -m gpu -k "10m" --durations=5 2>&1 | tail -8
