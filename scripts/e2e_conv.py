"""e2e of the conv extractor through qrm_detect_host (mode 0) per plan."""
import os, sys, time, json, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
base = q.DetectionConfig()
cfg = dataclasses.replace(base, extractor="conv")
B = 4096
pool = q.make_corpus(base, 1000, 2 * B)
host = torch.empty(pool.shape, dtype=torch.uint8, pin_memory=True); host.copy_(pool)
recs_pin = torch.empty((B, q.RECORD_DTYPE.itemsize), dtype=torch.uint8, pin_memory=True)
recs = recs_pin.numpy().view(q.RECORD_DTYPE).reshape(-1)
with q.DetectionContext(cfg) as ctx:
    for mb in (4096, 2048, 1024, 512):
        plan = ([1, 1, 1], [mb] * 3)
        for i in range(2):
            ctx.detect_host(None, i * B, plan=plan, mode=0, out=recs, ptr=host[(i % 2) * B].data_ptr(), shape=(B, 256, 256))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n = 4
        for i in range(n):
            ctx.detect_host(None, i * B, plan=plan, mode=0, out=recs, ptr=host[(i % 2) * B].data_ptr(), shape=(B, 256, 256))
        dt = time.perf_counter() - t0
        print(json.dumps({"mb": mb, "img_per_s": round(B * n / dt)}), flush=True)
    imgs = pool[:B]
    ctx.hidden_detect_device(imgs, logits=False); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(4): ctx.hidden_detect_device(imgs, logits=False)
    torch.cuda.synchronize()
    print(json.dumps({"device_only": round(4 * B / (time.perf_counter() - t0))}))
