"""configs[4] piece of bench.py alone: 1M images through detect_host (mode 0), calls of N."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
cfg = q.DetectionConfig()
pool = q.make_corpus(cfg, 1000, 8192)
host = torch.empty(pool.shape, dtype=torch.uint8, pin_memory=True); host.copy_(pool)
with q.DetectionContext(cfg) as ctx:
    for call, mb in ((8192, 4096), (8192, 2048), (4096, 2048), (8192, 8192)):
        recs = torch.empty((call, q.RECORD_DTYPE.itemsize), dtype=torch.uint8, pin_memory=True).numpy().view(q.RECORD_DTYPE).reshape(-1)
        ctx.detect_host(None, 0, plan=([1, 2, 1], [mb] * 3), mode=0, out=recs, ptr=host[0].data_ptr(), shape=(call, 256, 256))
        t0 = time.perf_counter()
        n = 0
        for first in range(0, 400_000, call):
            ctx.detect_host(None, first, plan=([1, 2, 1], [mb] * 3), mode=0, out=recs, ptr=host[0].data_ptr(), shape=(call, 256, 256))
            n += call
        print(json.dumps({"call": call, "mb": mb, "img_per_s": round(n / (time.perf_counter() - t0))}), flush=True)
