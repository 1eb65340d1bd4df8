"""Mode-0 host pipeline per tile size (512^2 images, 2048 per call): images/s and
window GB/s over PCIe, to see whether a tile size's transfer kernel keeps up."""
import dataclasses, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
n = 2048
out = {}
for l in (32, 64, 128):
    cfg = dataclasses.replace(q.DetectionConfig(), tile_size=l)
    d = q.make_corpus(cfg, 5000 + l, n, 512, 512)
    host = torch.empty(d.shape, dtype=torch.uint8, pin_memory=True)
    host.copy_(d)
    del d
    recs = torch.empty((n, q.RECORD_DTYPE.itemsize), dtype=torch.uint8, pin_memory=True).numpy().view(q.RECORD_DTYPE).reshape(-1)
    with q.DetectionContext(cfg) as ctx:
        for _ in range(2):
            ctx.detect_host(None, 0, plan=([1, 1, 1], [n] * 3), mode=0, out=recs, ptr=host.data_ptr(), shape=(n, 512, 512))
        t0 = time.perf_counter()
        for i in range(5):
            ctx.detect_host(None, i * n, plan=([1, 1, 1], [n] * 3), mode=0, out=recs, ptr=host.data_ptr(), shape=(n, 512, 512))
        dt = (time.perf_counter() - t0) / 5
    out[l] = {"img_per_s": round(n / dt), "window_GBps": round(n * 3 * l * l / dt / 1e9, 1), "verified": float(recs["verified"].mean())}
    del host
print(json.dumps(out))
