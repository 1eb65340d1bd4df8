"""Small workloads for compute-sanitizer (racecheck / synccheck / memcheck):
the decode kernel at split-K S = 1, 2, 4 (+ ties and the general-t completion
kernel), the conv pair kernels, the host executor in transfer modes 0-3, the
RS decoders (thread, segmented warp, codebook, symbols incl. the long-code
lane-parallel path) and the bf16 tile extraction. Each case checks its result
against the device path's own invariants (no oracle needed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_02447_b200 as q

case = sys.argv[1] if len(sys.argv) > 1 else "all"
cfg = q.DetectionConfig()
imgs = torch.cat([q.make_corpus(cfg, 1000, 96), q.make_corpus(cfg, 5000, 96, embed=False)]).contiguous()

if case in ("all", "decode"):
    for S in ("1", "2", "4"):
        os.environ["QRM_CORR_KSPLIT"] = S
        with q.DetectionContext(cfg) as ctx:
            rec = q.records_from_device(ctx.detect_device(imgs))
        torch.cuda.synchronize()
        assert rec["verified"][:96].all() and not rec["verified"][96:].any(), S
    os.environ.pop("QRM_CORR_KSPLIT")
    c2 = q.DetectionConfig(code=q.CodeParams.make(4, 15, 9))  # general t: completion kernel
    neg = q.make_corpus(c2, 7000, 64, embed=False)
    with q.DetectionContext(c2) as ctx:
        q.records_from_device(ctx.detect_device(neg))
    torch.cuda.synchronize()
    print("decode ok")

if case in ("all", "host"):
    host = imgs.cpu().numpy()
    with q.DetectionContext(cfg) as ctx:
        dev = q.records_from_device(ctx.detect_device(imgs))
        for mode in (0, 1, 2, 3):
            got, _ = ctx.detect_host(host, 0, plan=([1, 2, 1], [64] * 3), mode=mode)
            assert np.array_equal(got, dev), mode
    print("host ok")

if case in ("all", "conv"):
    with q.DetectionContext(cfg) as ctx:
        lg, rec = ctx.hidden_detect_device(imgs[:8], weight_seed=7, first_draw=0)
    torch.cuda.synchronize()
    assert torch.isfinite(lg).all()
    print("conv ok")

if case in ("all", "rs"):
    code = q.resolve_profile("gf16-15-12")
    _, words, ne_true = q.rs_stress_words(code, 5, 20000)
    outs = []
    for algo in (1, 2, 3):
        cw, ne = q.bw_decode_packed(code, words, algo=algo)
        outs.append((cw, ne))
    torch.cuda.synchronize()
    for cw, ne in outs[1:]:
        assert torch.equal(ne, outs[0][1])
    for mnk, n_words in (((8, 12, 8), 4000), ((8, 255, 223), 64), ((8, 100, 40), 64)):
        c = q.CodeParams.make(*mnk)
        tc, rv, nt = q.rs_stress_symbols(c, 3, n_words)
        cw, ne = q.bw_decode_symbols(c, rv)
        torch.cuda.synchronize()
        small = nt <= c.t
        assert torch.equal(cw[small], tc[small])
    print("rs ok")

if case in ("all", "tiles"):
    with q.DetectionContext(cfg) as ctx:
        t = ctx.extract_tiles(imgs[:64])
    torch.cuda.synchronize()
    print("tiles ok")
