"""Host executor per-call cost: wall time of qrm_detect_host (mode 0, pinned host
images, pinned records) against the call size; the intercept is the fixed cost."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_02447_b200 as q

cfg = q.DetectionConfig()
pool = q.make_corpus(cfg, 1000, 4096)
host = torch.empty(pool.shape, dtype=torch.uint8, pin_memory=True)
host.copy_(pool)
recs_pin = torch.empty((4096, q.RECORD_DTYPE.itemsize), dtype=torch.uint8, pin_memory=True)
recs = recs_pin.numpy().view(q.RECORD_DTYPE).reshape(-1)
res = {}
with q.DetectionContext(cfg) as ctx:
    for n in (16, 64, 256, 1024, 4096):
        plan = ([1, 2, 1], [n] * 3)
        for _ in range(5):
            ctx.detect_host(None, 0, plan=plan, mode=0, out=recs[:n], ptr=host.data_ptr(), shape=(n, 256, 256))
        ts = []
        for i in range(30):
            t0 = time.perf_counter()
            ctx.detect_host(None, i * n, plan=plan, mode=0, out=recs[:n], ptr=host.data_ptr(), shape=(n, 256, 256))
            ts.append((time.perf_counter() - t0) * 1e6)
        res[n] = round(float(np.median(ts)), 1)
print(json.dumps({"us_per_call_median": res}))
