cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_hidden.py tests/test_gpu_detect.py -x -q -m gpu > gpurun_out/t.log 2>&1; echo "tests rc=$?" >> gpurun_out/t.log; tail -3 gpurun_out/t.log
KS=0 timeout 120 python scripts/sweep_corr.py 2>&1 | grep -E "batch': (2048|4096|16384|65536)"
timeout 120 python scripts/bench_hidden.py 4096 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python scripts/bench_hidden.py 1024 2>/dev/null | grep -E "conv0" | head -3
