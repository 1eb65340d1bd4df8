cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_hidden.py tests/test_cpp_dropin.py -x -q -m gpu 2>&1 | tail -3
timeout 120 python scripts/debug_hidden_layers.py 2 2>&1 | tail -4
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --rs-words 1000000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['learned_extractor']))"
