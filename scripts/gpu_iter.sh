cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_hidden.py tests/test_cpp_dropin.py tests/test_gpu_detect.py -x -q -m gpu > gpurun_out/t.log 2>&1; echo "tests rc=$?" >> gpurun_out/t.log; grep -v "^  File" gpurun_out/t.log | tail -30
