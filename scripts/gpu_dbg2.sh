cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_hidden.py -x -q -m gpu -s > gpurun_out/hidden_test.log 2>&1; echo "rc=$?" >> gpurun_out/hidden_test.log
QRM_DEBUG_TIMES=1 timeout 300 python scripts/dbg_corr.py > gpurun_out/dbg.log 2>&1
KS=0 timeout 300 python scripts/sweep_corr.py > gpurun_out/sweep.log 2>&1
tail -5 gpurun_out/hidden_test.log; cat gpurun_out/dbg.log | grep qrm; cat gpurun_out/sweep.log
