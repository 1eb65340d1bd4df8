"""RS-only timing: 10M gf16-15-12 stress words through the t=1 and warp decoders."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
code = q.resolve_profile("gf16-15-12")
msg, words, ne_true = q.rs_stress_words(code, 2026, N)
cw = torch.empty_like(words)
ne = torch.empty(N, dtype=torch.int8, device=words.device)
out = {}
for algo in (1, 2):
    for _ in range(3):
        q.bw_decode_packed(code, words, cw, ne, algo=algo)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        q.bw_decode_packed(code, words, cw, ne, algo=algo)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    out[algo] = {"ms": ms, "Gcw_s": N / ms / 1e6, "GBs": 17 * N / ms / 1e6}
print(json.dumps(out))
