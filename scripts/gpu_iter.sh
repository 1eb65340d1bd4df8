cd $GRAFT_REPO_ROOT
QRM_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/b2.json 2> gpurun_out/b2.err; echo rc=$?
tail -5 gpurun_out/b2.err; python -c "import json; d=json.load(open('gpurun_out/b2.json')); print(d['n_gpus'], d['value'], d['e2e']['value'], d['config']['global_batch'], d['job_1m'])"
QRM_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/b2r.json 2> gpurun_out/b2r.err; echo rc=$?; head -c 300 gpurun_out/b2r.json
