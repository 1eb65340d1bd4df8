cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none --import-source on -k regex:corr_detect -s 4 -c 1 -o gpurun_out/corr_4k python scripts/profile_corr.py 4096 6 > gpurun_out/ncu4k.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv64 -s 10 -c 1 -o gpurun_out/conv64 python scripts/bench_hidden.py 1024 > gpurun_out/ncu_conv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv0 -s 2 -c 1 -o gpurun_out/conv0 python scripts/bench_hidden.py 1024 > gpurun_out/ncu_conv0.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fetch_windows -s 4 -c 1 -o gpurun_out/fetch python scripts/e2e_modes.py > gpurun_out/ncu_fetch.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_hidden.csv python scripts/bench_hidden.py 1024 > /dev/null 2>&1
tail -2 gpurun_out/ncu4k.log gpurun_out/ncu_conv.log gpurun_out/ncu_conv0.log gpurun_out/ncu_fetch.log; ls -la gpurun_out
