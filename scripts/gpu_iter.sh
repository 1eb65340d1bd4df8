cd $GRAFT_REPO_ROOT
( time timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err ) 2> gpurun_out/bench_time.txt
tail -3 gpurun_out/bench.err; grep real gpurun_out/bench_time.txt
python -c "
import json; d = json.load(open('gpurun_out/bench.json'))
for k in ('value','e2e','job_1m','tile_extract','config_512'): print(k, json.dumps(d.get(k))[:400])
"
