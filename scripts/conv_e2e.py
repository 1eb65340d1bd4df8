"""Learned-extractor end to end through qrm_detect_host: plans and transfer modes
(4096-image calls from pinned host memory) next to the device-resident batch."""
import dataclasses, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q

B = 4096
cfg = dataclasses.replace(q.DetectionConfig(), extractor="conv")
pool = q.make_corpus(q.DetectionConfig(), 1000, 2 * B)
host = torch.empty(pool.shape, dtype=torch.uint8, pin_memory=True)
host.copy_(pool)
recs_pin = torch.empty((B, q.RECORD_DTYPE.itemsize), dtype=torch.uint8, pin_memory=True)
recs = recs_pin.numpy().view(q.RECORD_DTYPE).reshape(-1)
out = {}
with q.DetectionContext(cfg) as ctx:
    for mb in (4096, 2048, 1024):
        dev = pool[:mb]
        for _ in range(2):
            ctx.hidden_detect_device(dev, logits=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            ctx.hidden_detect_device(dev, logits=False)
        torch.cuda.synchronize()
        out[f"device mb={mb}"] = mb * 3 / (time.perf_counter() - t0)
    for mode in (0, 2, 3):
        for plan in (([1, 1, 1], [4096] * 3), ([1, 2, 1], [2048] * 3), ([1, 2, 1], [1024] * 3), ([2, 2, 1], [1024] * 3)):
            def one(i):
                b0 = (i % 2) * B
                return ctx.detect_host(None, i * B, plan=plan, mode=mode, out=recs, ptr=host[b0].data_ptr(),
                                       shape=(B, 256, 256))
            one(0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(4):
                one(1 + i)
            out[f"mode {mode} plan {plan[0]} mb {plan[1][0]}"] = 4 * B / (time.perf_counter() - t0)
            print(json.dumps({k: round(v) for k, v in out.items()}), flush=True)
