cd $GRAFT_REPO_ROOT
timeout 600 python scripts/debug_hidden_layers.py 2 > gpurun_out/hidden_layers.log 2>&1; echo rc=$? >> gpurun_out/hidden_layers.log
cat gpurun_out/hidden_layers.log | tail -30
