cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu --timeout 400 > gpurun_out/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests.log
QRM_DEBUG_TIMES=1 python scripts/dbg_corr.py > gpurun_out/dbg.log 2>&1
KS=0 python scripts/sweep_corr.py > gpurun_out/sweep.log 2>&1
tail -4 gpurun_out/tests.log; grep "count=4096" gpurun_out/dbg.log | tail -8; grep "count=16384" gpurun_out/dbg.log | tail -8; cat gpurun_out/sweep.log
