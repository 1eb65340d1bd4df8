cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu1_smi.txt 2>&1
timeout 120 python __graft_entry__.py smoke > gpurun_out/gpu1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/gpu1_smoke.log
timeout 600 python -m pytest tests/test_gpu_rs.py tests/test_gpu_detect.py -x -q -m gpu --timeout 300 > gpurun_out/gpu1_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu1_tests.log
tail -5 gpurun_out/gpu1_smoke.log; tail -30 gpurun_out/gpu1_tests.log
