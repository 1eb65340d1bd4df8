"""The C++ drop-in's detect_batch e2e (tests/cpp/bench_dropin.cpp via bench.py's
dropin_submetric) plus mode-2 (host-staged windows) e2e through the C-ABI."""
import json, os, sys, time, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
import bench

cfg = q.DetectionConfig()
B = 4096
pool = q.make_corpus(cfg, 1000, B)
imgs = pool.cpu().numpy()
res = bench.dropin_submetric(imgs, types.SimpleNamespace(steps=50, warmup=3), 0)
print(json.dumps({k: res[k] for k in ("images_per_s", "ms_per_call_median", "desk_report_last")}))
