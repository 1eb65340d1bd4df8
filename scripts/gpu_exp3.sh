cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_hidden.py tests/test_gpu_detect.py -x -q -m gpu 2>&1 | tail -2
timeout 120 python scripts/bench_hidden.py 4096 2>&1 | tail -1
timeout 120 python scripts/bench_hidden.py 512 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/bench_hidden.py 512 2>/dev/null | grep -E "conv|hidden" | tail -10 | cut -d, -f5,15 > gpurun_out/hidden_launches.csv; cat gpurun_out/hidden_launches.csv
for f in 0 2; do QRM_EXP_FLAGS=$f KS=0 timeout 200 python scripts/sweep_corr.py 2>&1 | grep ksplit | tr '\n' ' '; echo; done
QRM_EXP_FLAGS=2 QRM_DEBUG_TIMES=1 timeout 120 python scripts/dbg_corr.py 2>&1 | grep "qrm dbg" | sed -n 9,16p
