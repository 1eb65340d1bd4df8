"""Host-side enqueue cost of one device-resident detect call vs the GPU step time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
cfg = q.DetectionConfig(); B = 4096
pool = q.make_corpus(cfg, 1000, 4 * B)
out = torch.empty((B, 24), dtype=torch.uint8, device="cuda")
views = [pool[i * B:(i + 1) * B] for i in range(4)]
with q.DetectionContext(cfg) as ctx:
    for i in range(20): ctx.detect_device(views[i % 4], i * B, out=out)
    torch.cuda.synchronize()
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 400
        a.record()
        t0 = time.perf_counter()
        for i in range(n): ctx.detect_device(views[i % 4], i * B, out=out)
        t1 = time.perf_counter()
        b.record(); torch.cuda.synchronize()
        print(f"host enqueue {(t1 - t0) / n * 1e6:.2f} us/call, gpu {a.elapsed_time(b) / n * 1e3:.2f} us/step", flush=True)
