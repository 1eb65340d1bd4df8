"""Edge cases of the device entry points: empty batches, single images, batch
sizes around the decode kernel's tile / split-K boundaries, and argument
errors (InvalidInput, never a crash or a silent fallback)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg(qrm):
    return qrm.DetectionConfig()


def test_empty_batches(qrm, cuda, cfg):
    empty = cuda.empty((0, 256, 256, 3), dtype=cuda.uint8, device="cuda")
    with qrm.DetectionContext(cfg) as ctx:
        assert qrm.records_from_device(ctx.detect_device(empty)).size == 0
        out, st = ctx.detect_host(np.zeros((0, 256, 256, 3), np.uint8), 0)
        assert out.size == 0 and st["minibatches"] == 0
        assert ctx.detect_ragged([]).size == 0
        assert ctx.extract_tiles(empty).shape == (0, 64, 64, 3)
        lg, rec = ctx.hidden_detect_device(empty)
        assert lg.shape[0] == 0 and rec.shape[0] == 0
    code = qrm.resolve_profile("gf16-15-12")
    cw, ne = qrm.bw_decode_packed(code, cuda.empty(0, dtype=cuda.int64, device="cuda"))
    assert cw.numel() == 0 and ne.numel() == 0
    assert qrm.apply_attack(empty, "blur", 1.0).shape == (0, 256, 256, 3)


@pytest.mark.parametrize("n", [1, 2, 15, 16, 17, 127, 128, 129, 1000, 4097])
def test_batch_size_boundaries(qrm, cuda, ref, cfg, n):
    """Images per decode tile (<= 128 TMEM lanes), tiles balanced over the SMs,
    split-K clusters of 1/2/4: records equal the reference for every size."""
    imgs = qrm.make_corpus(cfg, 3000, n)
    with qrm.DetectionContext(cfg) as ctx:
        rec = qrm.records_from_device(ctx.detect_device(imgs, first_draw=5))
    assert rec["verified"].all()
    host = imgs.cpu().numpy()
    # the reference numbers draws by position: image i of the batch is draw 5 + i
    for i in sorted({0, n // 2, n - 1}):
        Ri = ref.detect_sequential([host[i]], oracle.DetectCfg(), first_draw=5 + i)
        assert int(rec["raw"][i]) == oracle.bits_to_word(Ri["raw_bits"][0])
        assert int(rec["msg"][i]) == oracle.bits_to_word(Ri["corrected"][0])
        assert bool(rec["verified"][i]) == bool(Ri["verified"][0])


def test_argument_errors(qrm, cuda, cfg):
    imgs = qrm.make_corpus(cfg, 3000, 2)
    with qrm.DetectionContext(cfg) as ctx:
        with pytest.raises(qrm.InvalidInput):
            ctx.detect_device(imgs[:, :, :, :2].contiguous())  # 2 channels: stride smaller than an image
        with pytest.raises(qrm.InvalidInput):
            ctx.extract_tiles(imgs, channels=5)
        with pytest.raises(qrm.InvalidInput):
            ctx.detect_host(np.zeros((1, 256, 256, 3), np.uint8), 0, mode=7)
        with pytest.raises(qrm.InvalidInput):
            ctx.detect_host(np.zeros((1, 256, 256, 3), np.uint8), 0, plan=([1, 0, 1], [8, 8, 8]))
    with pytest.raises(qrm.InvalidInput):
        qrm.apply_attack(imgs, "crop", 2.0)
    with pytest.raises(qrm.InvalidInput):
        qrm.apply_attack(imgs, "nonsense", 1.0)
    small = qrm.DetectionConfig(tile_size=32)
    with qrm.DetectionContext(small) as ctx:
        with pytest.raises(qrm.InvalidInput):
            ctx.hidden_detect_device(imgs)  # the conv extractor is defined on 64x64 tiles
    import dataclasses
    with pytest.raises(qrm.InvalidInput):
        qrm.DetectionContext(dataclasses.replace(small, extractor="conv"))
