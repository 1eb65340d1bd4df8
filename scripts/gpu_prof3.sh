cd $GRAFT_REPO_ROOT
for ks in 1 2 4; do echo "== KS $ks"; KS=$ks python scripts/sweep_corr.py 2>&1 | grep -E "batch': (2048|4096|8192)"; done
ncu --set full --clock-control none --import-source on -k regex:corr_detect -s 4 -c 1 -o gpurun_out/corr_4k_v3 python scripts/profile_corr.py 4096 6 > gpurun_out/ncu4k.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:corr_detect -s 4 -c 1 -o gpurun_out/corr_64k_v3 python scripts/profile_corr.py 65536 6 > gpurun_out/ncu64k.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_v3.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --rs-words 1000000 > gpurun_out/bench_under_ncu.log 2>&1
tail -1 gpurun_out/ncu4k.log gpurun_out/ncu64k.log 2>/dev/null | head; wc -l gpurun_out/launches_v3.csv
