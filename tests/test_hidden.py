"""Learned extractor (HiDDeN-style conv stack; oracle/hidden_oracle.c is the contract).

Parity here is NOT pinned by the reference (it has no conv extractor,
SPEC.md:364): the C oracle is cross-checked against a plain PyTorch fp32
model built from the same parameters, and the sm_100a bf16 tensor-core path
against the oracle with a stated tolerance:
  * logits: relative L2 error <= 1e-2 (bf16 weights/activations, tf32 first layer, fp32 accumulate)
  * hard bits: equal wherever |logit_ref| > 0.1 * rms(logit_ref)
  * RS-corrected messages / verify: bit-exact given the GPU's own hard bits.
"""
import numpy as np
import pytest

import oracle

SEED = 7
NB = 60
REL_L2_TOL = 1e-2
NEAR_ZERO = 0.1


def _torch_forward(Ws, bns, wl, bl, tile_u8):
    import torch
    import torch.nn.functional as F
    x = torch.tensor((tile_u8.astype(np.float64) / 127.5 - 1.0).astype(np.float32)).permute(2, 0, 1)[None]
    for w, bn in zip(Ws, bns):
        cout, _, cin = w.shape
        k = torch.tensor(w).view(cout, 3, 3, cin).permute(0, 3, 1, 2).contiguous()
        y = F.conv2d(x, k, padding=1)
        g, b, m, v = (torch.tensor(a)[None, :, None, None] for a in bn)
        x = torch.relu((y - m) / torch.sqrt(v + 1e-5) * g + b)
    pooled = x.mean(dim=(2, 3))[0]
    return (torch.tensor(wl) @ pooled + torch.tensor(bl)).numpy()


def test_oracle_matches_torch_fp32(orc):
    Ws, bns, wl, bl = orc.hidden_params(SEED, NB)
    img = orc.make_corpus(1000, 1, 256, 256)[0]
    for (x, y) in [(0, 0), (64, 128)]:
        tile = np.ascontiguousarray(img[y:y + 64, x:x + 64])
        lg, _ = orc.hidden_forward(SEED, NB, tile)
        lt = _torch_forward(Ws, bns, wl, bl, tile)
        assert np.max(np.abs(lg - lt)) <= 1e-4 * max(1.0, np.max(np.abs(lt)))


@pytest.mark.gpu
def test_conv_extractor_matches_oracle(qrm, cuda, orc):
    cfg = qrm.DetectionConfig()
    imgs = cuda.cat([qrm.make_corpus(cfg, 1000, 6), qrm.make_corpus(cfg, 5000, 6, embed=False)])
    with qrm.DetectionContext(cfg) as ctx:
        lg, rec = ctx.hidden_detect_device(imgs, weight_seed=SEED, first_draw=3)
        cuda.cuda.synchronize()
    lg = lg.cpu().numpy().astype(np.float64)
    rec = qrm.records_from_device(rec)
    host = imgs.cpu().numpy()
    refs = []
    for i in range(host.shape[0]):
        x, y = orc.select_tile(256, 256, 64, "random_grid", 0, 3 + i)
        refs.append(orc.hidden_forward(SEED, NB, np.ascontiguousarray(host[i, y:y + 64, x:x + 64]))[0])
    ref = np.array(refs)
    rel = np.linalg.norm(lg - ref) / np.linalg.norm(ref)
    print(f"logit rel L2 = {rel:.3e}")
    assert rel <= REL_L2_TOL
    rms = np.sqrt(np.mean(ref ** 2))
    confident = np.abs(ref) > NEAR_ZERO * rms
    assert np.array_equal((lg > 0)[confident], (ref > 0)[confident])
    # hard bits of the record are the GPU logits' signs
    gpu_bits = np.array([oracle.bits_to_word((row > 0).astype(np.uint8)) for row in lg], np.uint64)
    assert np.array_equal(rec["raw"], gpu_bits)
    # RS + verify bit-exact on the GPU's own raw bits
    key = orc.default_message(1, 48)
    kcw = orc.rs_encode(4, 15, 12, key)
    for i in range(len(rec)):
        bits = oracle.word_to_bits(int(rec["raw"][i]), 60)
        res = orc.bw_decode(4, 15, 12, bits)
        assert (res is not None) == bool(rec["status"][i] == 1)
        matches = int((bits == kcw).sum())
        assert matches == int(rec["matches"][i])
        if res is not None:
            assert oracle.bits_to_word(res[0]) == int(rec["msg"][i]) and res[2] == int(rec["errors"][i])
            assert bool(rec["verified"][i]) == (int((res[0] == key).sum()) >= 41)
        else:
            assert bool(rec["verified"][i]) == (matches >= 49)


@pytest.mark.gpu
def test_conv_pair_variant_matches_single(qrm, cuda, monkeypatch):
    """The CTA-pair (cta_group::2, M=256) conv layer gives the same logits as the
    single-CTA layer: identical bf16 products, fp32 accumulation in the same
    tap/K order per output pixel; the pair path's fused linear layer sums the
    logits in another order, so they agree to fp32 rounding."""
    cfg = qrm.DetectionConfig()
    imgs = cuda.cat([qrm.make_corpus(cfg, 1000, 40), qrm.make_corpus(cfg, 5000, 40, embed=False)])
    out = {}
    for pair in ("0", "1"):
        monkeypatch.setenv("QRM_CONV_PAIR", pair)
        with qrm.DetectionContext(cfg) as ctx:
            lg, rec = ctx.hidden_detect_device(imgs, weight_seed=SEED, first_draw=11)
            cuda.cuda.synchronize()
        out[pair] = (lg.cpu().numpy(), qrm.records_from_device(rec))
    a, b = out["0"][0], out["1"][0]
    # the pair kernel's last layer also folds the linear layer into its epilogue
    # (fixed-point partial logits per block), so logits agree to fp32 rounding
    assert np.max(np.abs(a - b)) <= 1e-5 * max(1.0, np.max(np.abs(a)))
    sure = np.abs(a) > 1e-4 * np.max(np.abs(a))  # hard bits away from the fp32 noise
    def bits(r):  # packed raw word (bit o at word bit nbits-1-o) -> [n, nbits]
        b = np.ascontiguousarray(r["raw"]).astype("<u8").view(np.uint8).reshape(-1, 8)[:, ::-1]
        return np.unpackbits(b, axis=1)[:, 64 - a.shape[1]:]
    ra, rb = bits(out["0"][1]), bits(out["1"][1])
    assert np.array_equal(ra[sure], rb[sure])


@pytest.mark.gpu
def test_conv_extractor_through_detect_entry_points(qrm, cuda):
    """DetectionConfig(extractor="conv") routes detect_device / detect_host (all
    three transfer modes) through the conv stack; records equal the direct call."""
    import dataclasses
    base = qrm.DetectionConfig()
    cfg = dataclasses.replace(base, extractor="conv", conv_seed=SEED)
    imgs = cuda.cat([qrm.make_corpus(base, 1000, 20), qrm.make_corpus(base, 5000, 20, embed=False)])
    with qrm.DetectionContext(base) as ctx:
        _, rec0 = ctx.hidden_detect_device(imgs, weight_seed=SEED, first_draw=5, logits=False)
        ref = qrm.records_from_device(rec0)
    host = imgs.cpu().numpy()
    with qrm.DetectionContext(cfg) as ctx:
        dev = qrm.records_from_device(ctx.detect_device(imgs, first_draw=5))
        assert np.array_equal(dev, ref)
        for mode in (0, 1, 2):
            out, st = ctx.detect_host(host, 5, plan=([1, 2, 1], [16, 16, 16]), mode=mode)
            assert np.array_equal(out, ref), mode
        rag = ctx.detect_ragged(list(host), first_draw=5)  # staged-window path
        assert np.array_equal(rag, ref)
    with pytest.raises(qrm.InvalidInput):
        qrm.DetectionContext(dataclasses.replace(base, extractor="cnn"))
