"""Small driver for ncu: a few device-resident detect launches (batch 4096)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = q.DetectionConfig()
imgs = q.make_corpus(cfg, 1000, batch * 2)
with q.DetectionContext(cfg) as ctx:
    for i in range(reps):
        ctx.detect_device(imgs[(i % 2) * batch:(i % 2 + 1) * batch], first_draw=i * batch)
    torch.cuda.synchronize()
print("done")
