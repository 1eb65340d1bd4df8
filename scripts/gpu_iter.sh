cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 10 --no-cpu-baseline --rs-words 1000000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['tile_extract']))"
ncu --set full --clock-control none -k regex:tile_bf16 -s 2 -c 1 -o gpurun_out/tile_bf16 python bench.py --steps 3 --no-cpu-baseline --rs-words 100000 > /dev/null 2>&1; ls gpurun_out/tile_bf16*
