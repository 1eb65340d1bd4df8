"""Conv-extractor timing: per-layer kernel time and tensor throughput."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = q.DetectionConfig()
imgs = q.make_corpus(cfg, 1000, B)
flop_per_tile = 2 * 4096 * (27 * 64 + 7 * 576 * 64 + 576 * 60) + 2 * 60 * 60
with q.DetectionContext(cfg) as ctx:
    for _ in range(3):
        ctx.hidden_detect_device(imgs, logits=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record()
    for _ in range(reps):
        ctx.hidden_detect_device(imgs, logits=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
print(json.dumps({"tiles": B, "ms": ms, "tiles_per_s": B / ms * 1e3, "TFLOPs": flop_per_tile * B / ms / 1e9}))
