cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
free -g > gpurun_out/r2b_free.txt
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -x -s -k "parity_scale or dropin" > gpurun_out/r2b_new.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_new.log
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/r2b_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2b_tests.log
timeout 600 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
tail -5 gpurun_out/r2b_new.log; tail -3 gpurun_out/r2b_tests.log; tail -2 gpurun_out/r2b_bench.err; head -c 600 gpurun_out/r2b_bench.json
