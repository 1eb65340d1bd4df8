"""ncu driver: one decode launch on a clean batch, then one on an unwatermarked batch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
B = 4096
cfg = q.DetectionConfig()
clean = q.make_corpus(cfg, 1000, B)
neg = q.make_corpus(cfg, 90000, B, embed=False)
with q.DetectionContext(cfg) as ctx:
    for i in range(3):
        ctx.detect_device(clean, first_draw=0)
    ctx.detect_device(clean, first_draw=0)
    ctx.detect_device(neg, first_draw=0)
    torch.cuda.synchronize()
print("done")
