"""Robustness attacks on the device: apply_attack
(transforms.cpp:289-362) bit-exact with the compiled reference for every
TransformOp, on ragged sizes (odd widths, partial JPEG blocks), plus the
attack_suite detection sweep (the paper's Table 3 analogue) against the
reference pipeline's records."""
import numpy as np
import pytest

import oracle

OPS = [("centercrop", 200), ("centercrop", 1000), ("resizeto", 97), ("resizeto", 300), ("normalize", 0.0),
       ("crop", 0.1), ("crop", 0.5), ("crop", 1.0), ("resize", 0.5), ("resize", 0.37), ("resize", 1.0),
       ("brightness", 2.0), ("brightness", 0.3), ("brightness", 1.0), ("contrast", 2.0), ("contrast", 0.5),
       ("saturation", 0.0), ("saturation", 1.7), ("sharpness", 2.0), ("sharpness", 0.0), ("blur", 1.0),
       ("overlay_text", 0.0), ("jpeg_approx", 50.0), ("jpeg_approx", 10.0), ("jpeg_approx", 95.0),
       ("jpeg_approx", 100.0)]

BAD = [("centercrop", 0), ("resizeto", -3), ("crop", 0.0), ("crop", 1.5), ("resize", 1.2), ("resize", 0.0),
       ("brightness", -1.0), ("contrast", -0.1), ("saturation", -2.0), ("sharpness", -1.0), ("jpeg_approx", 0.0),
       ("jpeg_approx", 101.0)]


def test_attack_argument_errors_match_reference(qrm, ref):
    """Checks and messages are host-side: no GPU needed to compare them."""
    import ctypes as C
    img = np.zeros((16, 16, 3), np.uint8)
    for op, p in BAD:
        with pytest.raises(ValueError) as want:
            ref.apply_attack(img, op, p)
        ow, oh = C.c_int(), C.c_int()
        rc = qrm.lib().qrm_attack_device(None, 1, 16, 16, 16 * 16 * 3, qrm.ATTACKS.index(op), p, None, 0,
                                         C.byref(ow), C.byref(oh), None)
        assert rc == 1 and qrm.lib().qrm_last_error().decode() == str(want.value), (op, p)


@pytest.mark.gpu
def test_attacks_bit_exact_with_reference(qrm, ref, cuda):
    rng = np.random.default_rng(5)
    cfg = qrm.DetectionConfig()
    for (h, w) in [(256, 256), (61, 83), (300, 171)]:
        base = qrm.make_corpus(cfg, 1000, 2, w, h).cpu().numpy()
        noise = rng.integers(0, 256, (1, h, w, 3), dtype=np.uint8)
        flat = np.full((1, h, w, 3), 77, np.uint8)
        host = np.concatenate([base, noise, flat])
        dev = cuda.tensor(host, device="cuda")
        for op, p in OPS:
            got = qrm.apply_attack(dev, op, p).cpu().numpy()
            for i in range(host.shape[0]):
                want = ref.apply_attack(host[i], op, p)
                assert got[i].shape == want.shape, (op, p, h, w)
                assert np.array_equal(got[i], want), (op, p, h, w, i, int((got[i] != want).sum()))


@pytest.mark.gpu
def test_attack_suite_detection_matches_reference(qrm, ref, cuda):
    """Detection after each attack of attack_suite: GPU attack + GPU detect gives
    the reference pipeline's records (semantic_equal fields)."""
    cfg = qrm.DetectionConfig()
    imgs = qrm.make_corpus(cfg, 1000, 12)
    for name, op, p in qrm.ATTACK_SUITE:
        att = qrm.apply_attack(imgs, op, p)
        with qrm.DetectionContext(cfg) as ctx:
            rec, _ = ctx.detect_host(att.cpu().numpy(), 0, mode=2)
        got = qrm.semantic_fields(rec, cfg.code)
        host = [ref.apply_attack(x, op, p) for x in imgs.cpu().numpy()]
        arrs, _ = ref.detect_batch(host, oracle.DetectCfg())
        raw = np.array([oracle.bits_to_word(b) for b in arrs["raw_bits"]], np.uint64)
        assert np.array_equal(got["raw"], raw), name
        assert np.array_equal(got["verified"], arrs["verified"].astype(bool)), name
        assert np.array_equal(got["decoded"], arrs["has_corrected"].astype(bool)), name
