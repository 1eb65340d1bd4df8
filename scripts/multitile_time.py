"""configs[2] multi-tile interleaving throughput (grouped page-locked path) vs
task size and stream count; 2048 images of 512^2, sizes 32/64/128 a third each."""
import dataclasses, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
from paper_2509_02447_b200.multitile import MultiTileDetector

cfg = q.DetectionConfig()
n = 2048
per = {32: n // 3, 64: n // 3, 128: n - 2 * (n // 3)}
pins, groups = [], {}
for l, cnt in per.items():
    d = q.make_corpus(dataclasses.replace(cfg, tile_size=l), 300000 + l, cnt, 512, 512)
    b = torch.empty(d.shape, dtype=torch.uint8, pin_memory=True)
    b.copy_(d)
    pins.append(b)
    groups[l] = (b.data_ptr(), cnt)
out = {}
for streams in (1, 2, 3):
    with MultiTileDetector(cfg, streams=streams) as mt:
        mt.warmup([pins[1][i].numpy() for i in range(256)], iters=2, b0=256)
        for mb in (256, 512, 1024):
            mt.detect_grouped(groups, (512, 512), minibatch=mb)
            t0 = time.perf_counter()
            for _ in range(4):
                recs, info = mt.detect_grouped(groups, (512, 512), minibatch=mb)
            out[f"streams {streams} mb {mb}"] = round(4 * n / (time.perf_counter() - t0))
            print(json.dumps(out), flush=True)
