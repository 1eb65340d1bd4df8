"""Decode-kernel sweep: back-to-back and isolated per-launch time of
detect_device at several batch sizes and split-K settings (QRM_CORR_KSPLIT, read
at context creation). Inputs rotate over a 16,384-image pool (> L2)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q

cfg = q.DetectionConfig()
pool = q.make_corpus(cfg, 1000, 16384)
big = None
res = []
splits = sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "1", "2", "4"]
batches = [int(b) for b in sys.argv[2].split(",")] if len(sys.argv) > 2 else [4096]
for S in splits:
    os.environ["QRM_CORR_KSPLIT"] = S
    with q.DetectionContext(cfg) as ctx:
        ctx.set_input_overlap(True)
        for B in batches:
            src = pool if B <= 16384 else pool.repeat(B // 16384, 1, 1, 1)
            nb = src.shape[0] // B
            views = [src[i * B:(i + 1) * B] for i in range(nb)]
            out = torch.empty((B, q.RECORD_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
            for i in range(5):
                ctx.detect_device(views[i % nb], first_draw=i * B, out=out)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(20, 200 * 4096 // B)
            a.record()
            for i in range(reps):
                ctx.detect_device(views[i % nb], first_draw=i * B, out=out)
            b.record()
            torch.cuda.synchronize()
            b2b = a.elapsed_time(b) / reps
            iso = []
            for i in range(10):
                a.record()
                ctx.detect_device(views[i % nb], first_draw=i * B, out=out)
                b.record()
                torch.cuda.synchronize()
                iso.append(a.elapsed_time(b))
            iso.sort()
            rec = q.records_from_device(out)
            assert rec["verified"].all()
            gbs = B * 12312 / (b2b / 1e3) / 1e9
            res.append({"ksplit": S, "batch": B, "b2b_us": b2b * 1e3, "iso_us_median": iso[5] * 1e3,
                        "b2b_GBs": gbs, "b2b_frac": gbs / 6552.3,
                        "iso_frac": B * 12312 / (iso[5] / 1e3) / 1e9 / 6552.3})
            print(json.dumps(res[-1]), flush=True)
        if big is not None:
            del big
