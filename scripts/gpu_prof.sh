cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none --import-source on -k regex:corr_detect -s 3 -c 1 -o gpurun_out/corr_full python scripts/profile_corr.py 4096 5 > gpurun_out/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --rs-words 1000000 > gpurun_out/bench_under_ncu.log 2>&1
tail -3 gpurun_out/ncu_full.log
