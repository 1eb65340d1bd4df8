cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_rs.py -x -q -m gpu 2>&1 | tail -2
timeout 120 python scripts/rs_time.py 2>&1 | tail -1
ncu --set full --clock-control none -k regex:rs_t1_packed_x4 -s 3 -c 1 -o gpurun_out/rs_t1 python scripts/rs_time.py > gpurun_out/ncu_rs.log 2>&1; tail -1 gpurun_out/ncu_rs.log
QRM_DEBUG_TIMES=1 timeout 120 python scripts/dbg_corr.py 2>&1 | grep "qrm dbg" > gpurun_out/corr_timeline.txt; cat gpurun_out/corr_timeline.txt
