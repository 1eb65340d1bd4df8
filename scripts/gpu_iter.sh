cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_formats.py tests/test_cpp_dropin.py tests/test_hidden.py tests/test_gpu_detect.py -x -q -m gpu 2>&1 | tail -3
