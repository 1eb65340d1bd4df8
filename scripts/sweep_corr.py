"""Decode-kernel scaling sweep: batch size x split-K -> kernel time and GB/s."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q

cfg = q.DetectionConfig()
pool = q.make_corpus(cfg, 1000, 65536)
res = []
with q.DetectionContext(cfg) as ctx:
    for ks in os.environ.get("KS", "0,1,2,4").split(","):
        if ks == "0":
            os.environ.pop("QRM_CORR_KSPLIT", None)
        else:
            os.environ["QRM_CORR_KSPLIT"] = ks
        for b in (128, 512, 1024, 2048, 4096, 8192, 16384, 65536):
            ms = ctx.kernel_time_probe(pool[:b], reps=10)
            gbs = b * 12288 / (ms / 1e3) / 1e9
            res.append({"ksplit": ks, "batch": b, "us": round(ms * 1e3, 2), "GBps": round(gbs, 1)})
            print(res[-1], flush=True)
json.dump(res, open(os.path.join(os.environ.get("OUT", "gpurun_out"), "sweep_corr.json"), "w"))
