"""e2e (host buffers -> host records) throughput of qrm_detect_host per mode and plan."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_02447_b200 as q
cfg = q.DetectionConfig()
B = 4096
pool = q.make_corpus(cfg, 1000, 4 * B)
host = torch.empty(pool.shape, dtype=torch.uint8, pin_memory=True); host.copy_(pool)
recs_pinned = torch.empty((B, q.RECORD_DTYPE.itemsize), dtype=torch.uint8, pin_memory=True)
recs = recs_pinned.numpy().view(q.RECORD_DTYPE).reshape(-1)
with q.DetectionContext(cfg) as ctx:
    modes = [int(m) for m in os.environ.get("E2E_MODES", "0,2,1").split(",")]
    fracs = [float(f) for f in os.environ.get("E2E_FRACS", "0.5").split(",")]
    for mode, frac in [(m, f) for m in modes for f in (fracs if m == 3 else [None])]:
        if frac is not None:
            ctx.set_transfer_split(frac)
        for streams, mb in (([1, 2, 1], 2048), ([1, 2, 1], 1024), ([2, 2, 2], 1024), ([1, 1, 1], 4096)):
            plan = (streams, [mb] * 3)
            def step(i):
                b = i % 4
                ctx.detect_host(None, i * B, plan=plan, mode=mode, out=recs, ptr=host[b * B].data_ptr(), shape=(B, 256, 256))
            for i in range(3): step(i)
            n = 12
            t0 = time.perf_counter()
            for i in range(n): step(3 + i)
            dt = time.perf_counter() - t0
            assert recs["verified"].all()
            print(json.dumps({"mode": mode, "frac": frac, "streams": streams, "mb": mb, "img_per_s": round(B * n / dt)}), flush=True)
