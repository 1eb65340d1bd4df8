"""Decode step time (device-resident, back to back, batch 4096) per corpus kind:
clean watermarked, blurred watermarked (RS corrections), unwatermarked (RS
failures + exact-zero ties), and the bench's mixed corpus."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q

B = 4096
cfg = q.DetectionConfig()
kinds = {
    "clean": [q.make_corpus(cfg, 1000 + b * B, B) for b in range(4)],
    "blurred": [q.apply_attack(q.make_corpus(cfg, 30000 + b * B, B), "blur", 1.0) for b in range(4)],
    "unwatermarked": [q.make_corpus(cfg, 90000 + b * B, B, embed=False) for b in range(4)],
}
out = torch.empty((B, q.RECORD_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
res = {}
with q.DetectionContext(cfg) as ctx:
    ctx.set_input_overlap(True)
    for name, bs in kinds.items():
        for i in range(5):
            ctx.detect_device(bs[i % 4], first_draw=i * B, out=out)
        torch.cuda.synchronize()
        rec = q.records_from_device(out)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(200):
            ctx.detect_device(bs[i % 4], first_draw=i * B, out=out)
        b.record()
        torch.cuda.synchronize()
        res[name] = {"us_per_step": a.elapsed_time(b) / 200 * 1e3, "ties": int((rec["ties"] > 0).sum()),
                     "failed": int((rec["status"] == 0).sum()), "corrected": int(((rec["status"] == 1) & (rec["errors"] > 0)).sum())}
        print(json.dumps({name: res[name]}), flush=True)
