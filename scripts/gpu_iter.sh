cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_hidden.py tests/test_cpp_dropin.py -x -q -m gpu 2>&1 | tail -2
for i in 1 2 3; do python scripts/bench_hidden.py 4096; done
ncu --set full --import-source on --clock-control none -k regex:conv64 -s 10 -c 1 -o gpurun_out/conv64pair2 python scripts/bench_hidden.py 1024 > /dev/null 2>&1; ls gpurun_out/conv64pair2*
