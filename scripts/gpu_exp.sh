cd $GRAFT_REPO_ROOT
KS=0 python scripts/sweep_corr.py > gpurun_out/exp_base.log 2>&1
QRM_EXP_FLAGS=1 KS=0 python scripts/sweep_corr.py > gpurun_out/exp_nofence.log 2>&1
QRM_EXP_FLAGS=1 timeout 300 python -m pytest tests/test_gpu_detect.py -x -q -m gpu > gpurun_out/exp_nofence_tests.log 2>&1
KS=1,4 python scripts/sweep_corr.py > gpurun_out/exp_ks.log 2>&1
tail -8 gpurun_out/exp_base.log; tail -8 gpurun_out/exp_nofence.log; tail -3 gpurun_out/exp_nofence_tests.log; cat gpurun_out/exp_ks.log
