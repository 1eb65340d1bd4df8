# Full GPU pass: tests, smoke, bench (both arms), ncu launch list + full captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 500 > gpurun_out/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --rs-words 1000000 > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:corr_detect -s 4 -c 1 -o gpurun_out/corr_4k python scripts/profile_corr.py 4096 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv64 -s 10 -c 1 -o gpurun_out/conv64 python scripts/bench_hidden.py 1024 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv64 -s 7 -c 1 -o gpurun_out/conv64_last python scripts/bench_hidden.py 1024 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv0 -s 2 -c 1 -o gpurun_out/conv0 python scripts/bench_hidden.py 1024 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fetch_windows -s 4 -c 1 -o gpurun_out/fetch python scripts/e2e_modes.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rs_t1_packed -s 3 -c 1 -o gpurun_out/rs_t1 python scripts/rs_time.py > /dev/null 2>&1
bash scripts/sanitize.sh > /dev/null 2>&1
tail -3 gpurun_out/tests.log; cat gpurun_out/sanitize_summary.txt; tail -1 gpurun_out/smoke.log; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json gpurun_out/bench_ref.json; ls gpurun_out
