"""Row f1 measurement: the general-t packed decoder with and without the device
codebook (algo 3 vs algo 2 of qrm_rs_decode_packed_device) on a 90 %-duplicate
stream: 10M words drawn from 1M distinct stress words. Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_02447_b200 as q

N, U = 10_000_000, 1_000_000
out = {"stream": f"{N:,} words drawn uniformly from {U:,} distinct stress words (~90% repeats)"}
for name, code in (("gf16-15-12 (t=1)", q.resolve_profile("gf16-15-12")), ("gf16 (15,11) (t=2)", q.CodeParams.make(4, 15, 11)),
                   ("gf16 (15,7) (t=4)", q.CodeParams.make(4, 15, 7))):
    _, uniq, _ = q.rs_stress_words(code, 4242, U)
    g = torch.Generator(device="cuda").manual_seed(1)
    idx = torch.randint(0, U, (N,), device="cuda", generator=g)
    words = uniq[idx].contiguous()
    res = {}
    ref_cw = ref_ne = None
    for algo in ((1, 2, 3) if code.t == 1 else (2, 3)):
        cw = torch.empty_like(words)
        ne = torch.empty(N, dtype=torch.int8, device="cuda")
        if algo == 3:
            q.rs_codebook_clear(code)
        q.bw_decode_packed(code, words, cw, ne, algo=algo)  # (algo 3: fills the codebook)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        a.record()
        for _ in range(reps):
            q.bw_decode_packed(code, words, cw, ne, algo=algo)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        if ref_cw is None:
            ref_cw, ref_ne = cw.clone(), ne.clone()
        assert torch.equal(ne, ref_ne) and torch.equal(cw[ne >= 0], ref_cw[ne >= 0])
        res[{1: "thread_t1", 2: "seg_warp_bm", 3: "seg_warp_bm + codebook"}[algo]] = {
            "ms": ms, "G_words_per_s": N / ms / 1e6}
    # cold codebook: the first pass over the stream inserts every distinct word
    q.rs_codebook_clear(code)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    q.bw_decode_packed(code, words, cw, ne, algo=3)
    b.record()
    torch.cuda.synchronize()
    res["seg_warp_bm + codebook (cold, first pass)"] = {"ms": a.elapsed_time(b), "G_words_per_s": N / a.elapsed_time(b) / 1e6}
    out[name] = res
print(json.dumps(out))
