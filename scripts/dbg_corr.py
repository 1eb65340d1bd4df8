import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
cfg = q.DetectionConfig()
pool = q.make_corpus(cfg, 1000, 16384)
with q.DetectionContext(cfg) as ctx:
    for b in (512, 512, 4096, 4096, 16384, 16384):
        ctx.detect_device(pool[:b])
        torch.cuda.synchronize()
