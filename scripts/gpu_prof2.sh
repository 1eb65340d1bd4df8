cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none --import-source on -k regex:corr_detect -s 4 -c 1 -o gpurun_out/corr_16k python scripts/profile_corr.py 16384 6 > gpurun_out/ncu16k.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:corr_detect -s 4 -c 1 -o gpurun_out/corr_4k python scripts/profile_corr.py 4096 6 > gpurun_out/ncu4k.log 2>&1
tail -2 gpurun_out/ncu16k.log gpurun_out/ncu4k.log
