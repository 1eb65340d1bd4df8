"""configs[2] through qrm_detect_host_lpt (Algorithm 2 placing mini-batches on decode
streams): e2e img/s per (plan, lambda, b_min) on 2048-image calls of 512^2."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
cfg = q.DetectionConfig()
n = 2048
d = q.make_corpus(cfg, 100000, n, 512, 512)
host = torch.empty(d.shape, dtype=torch.uint8, pin_memory=True)
host.copy_(d)
del d
recs = torch.empty((n, q.RECORD_DTYPE.itemsize), dtype=torch.uint8, pin_memory=True).numpy().view(q.RECORD_DTYPE).reshape(-1)
out = {}
with q.DetectionContext(cfg) as ctx:
    ctx.warmup_profile(iters=3, b0=16, mode=0, ptr=host.data_ptr(), shape=(n, 512, 512))
    for plan, lpt in ((([2, 2, 1], [512] * 3), (0.2, 128)), (([2, 2, 1], [512] * 3), (float("inf"), 128)),
                      (([1, 2, 1], [1024] * 3), (0.5, 256)), (([1, 2, 1], [1024] * 3), (float("inf"), 256)),
                      (([1, 1, 1], [2048] * 3), None)):
        for _ in range(2):
            ctx.detect_host(None, 0, plan=plan, mode=0, out=recs, ptr=host.data_ptr(), shape=(n, 512, 512), lpt=lpt)
        t0 = time.perf_counter()
        for i in range(8):
            ctx.detect_host(None, i * n, plan=plan, mode=0, out=recs, ptr=host.data_ptr(), shape=(n, 512, 512), lpt=lpt)
        out[f"{plan[0]} mb {plan[1][0]} lpt {lpt}"] = round(8 * n / (time.perf_counter() - t0))
        assert recs["verified"].all()
print(json.dumps(out))
