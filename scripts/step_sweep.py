"""Back-to-back device-resident decode steps (as bench.py's timed loop): per-step
time and window GB/s per batch size and split-K (QRM_CORR_KSPLIT)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
cfg = q.DetectionConfig()
pool = q.make_corpus(cfg, 1000, 65536)
res = []
with q.DetectionContext(cfg) as ctx:
    for b in (1024, 4096, 16384, 65536):
        for ks in ("", "1", "2", "4"):
            if ks: os.environ["QRM_CORR_KSPLIT"] = ks
            else: os.environ.pop("QRM_CORR_KSPLIT", None)
            nb = 65536 // b
            out = torch.empty((b, 24), dtype=torch.uint8, device="cuda")
            for i in range(5): ctx.detect_device(pool[(i % nb) * b:(i % nb + 1) * b], i * b, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 40
            e0.record()
            for i in range(n): ctx.detect_device(pool[(i % nb) * b:(i % nb + 1) * b], i * b, out=out)
            e1.record(); torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / n * 1e3
            res.append({"batch": b, "ksplit": ks or "auto", "us_per_step": round(us, 2),
                        "Mimg_s": round(b / us, 1), "GBps": round(b * 12312 / us / 1e3, 1)})
            print(json.dumps(res[-1]), flush=True)
