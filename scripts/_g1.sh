cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
lscpu > gpurun_out/r2a_lscpu.txt; numactl -H > gpurun_out/r2a_numa.txt 2>&1; nvidia-smi topo -m >> gpurun_out/r2a_numa.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu --timeout 500 -x > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2a_tests.log
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
tail -3 gpurun_out/r2a_tests.log; tail -2 gpurun_out/r2a_bench.err; cat gpurun_out/r2a_bench.json
