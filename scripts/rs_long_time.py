"""Long GF(2^8) code timing: (255,223) t=16 and (255,200) t=27 stress words through the segmented decoder."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q
out = {}
for mnk, n_words in (((8, 255, 223), 400_000), ((8, 255, 200), 100_000), ((8, 12, 8), 4_000_000)):
    code = q.CodeParams.make(*mnk)
    tc, rv, nt = q.rs_stress_symbols(code, 5, n_words)
    cw, ne = torch.empty_like(rv), torch.empty(n_words, dtype=torch.int8, device="cuda")
    for _ in range(2):
        q.bw_decode_symbols_into(code, rv, cw, ne)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        q.bw_decode_symbols_into(code, rv, cw, ne)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    small = nt <= code.t
    assert torch.equal(cw[small], tc[small])
    out[str(mnk)] = {"ms": ms, "M_cw_s": n_words / ms / 1e3}
print(json.dumps(out))
