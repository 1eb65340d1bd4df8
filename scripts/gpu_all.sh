cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu --timeout 500 > gpurun_out/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 120 python scripts/bench_hidden.py 4096 > gpurun_out/hidden_bench.log 2>&1
tail -15 gpurun_out/tests.log; tail -3 gpurun_out/smoke.log; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json gpurun_out/bench_ref.json; tail -3 gpurun_out/hidden_bench.log
