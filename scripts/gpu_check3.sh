cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu --timeout 400 > gpurun_out/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests.log
KS=0 python scripts/sweep_corr.py > gpurun_out/sweep.log 2>&1
QRM_DEBUG_TIMES=1 python scripts/dbg_corr.py > gpurun_out/dbg.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -4 gpurun_out/tests.log; cat gpurun_out/sweep.log; grep "count=4096" gpurun_out/dbg.log | tail -8; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
