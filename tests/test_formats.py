"""Ingest and report formats either side of the path:
PPM P6 I/O against the reference's read_ppm / write_ppm (image.cpp:106-156)
and the records JSON against the reference's record_to_json + nlohmann
dump(2) (json_io.cpp:98-120, cli.cpp:279-281)."""
import os

import numpy as np
import pytest

import oracle


@pytest.fixture(scope="module")
def ref():
    if not oracle.Reference.available():
        pytest.skip("compiled reference unavailable")
    return oracle.Reference()


def _noise(seed, h, w):
    return np.random.default_rng(seed).integers(0, 256, (h, w, 3), dtype=np.uint8)


def test_ppm_round_trip_both_directions(qrm, ref, tmp_path):
    for i, (h, w) in enumerate([(1, 1), (7, 13), (256, 256), (300, 200)]):
        img = _noise(i, h, w)
        a, b = tmp_path / f"a{i}.ppm", tmp_path / f"b{i}.ppm"
        qrm.write_ppm(img, a)
        ref.write_ppm(img, b)
        assert a.read_bytes() == b.read_bytes()  # byte-identical files
        assert np.array_equal(qrm.read_ppm(b), img)
        assert np.array_equal(ref.read_ppm(a), img)


def test_ppm_header_grammar_and_errors_match_reference(qrm, ref, tmp_path):
    raster = _noise(9, 3, 4).tobytes()
    cases = {
        "comments.ppm": b"P6\n# made by hand\n4 # width\n3\n# maxval next\n255\n" + raster,
        "tabs.ppm": b"P6\t4\r\n3  255 " + raster,
        "magic.ppm": b"P3\n4 3\n255\n" + raster,
        "maxval.ppm": b"P6\n4 3\n65535\n" + raster,
        "truncated.ppm": b"P6\n4 3\n255\n" + raster[:-5],
        "header.ppm": b"P6\n4 x\n255\n" + raster,
        "empty.ppm": b"",
    }
    for name, data in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        try:
            want = ref.read_ppm(p)
            err = None
        except ValueError as e:
            want, err = None, str(e)
        if err is None:
            assert np.array_equal(qrm.read_ppm(p), want), name
        else:
            with pytest.raises(qrm.InvalidInput) as ei:
                qrm.read_ppm(p)
            assert str(ei.value) == err, name
    with pytest.raises(qrm.InvalidInput, match="cannot open"):
        qrm.read_ppm(tmp_path / "missing.ppm")


def test_ppm_batch_ingest(qrm, tmp_path):
    imgs = [_noise(100 + i, 32, 48) for i in range(9)]
    paths = []
    for i, im in enumerate(imgs):
        paths.append(tmp_path / f"{i:03d}.ppm")
        qrm.write_ppm(im, paths[-1])
    out = qrm.read_ppm_batch(paths, threads=4)
    assert np.array_equal(out, np.stack(imgs))
    qrm.write_ppm(_noise(1, 10, 10), tmp_path / "odd.ppm")
    with pytest.raises(qrm.InvalidInput, match="size differs"):
        qrm.read_ppm_batch(paths + [tmp_path / "odd.ppm"])


def _pack(qrm, arrs, kcw):
    """Reference records (BitVec fields) -> the ABI record layout."""
    n = len(arrs["errors"])
    rec = np.zeros(n, dtype=qrm.RECORD_DTYPE)
    for i in range(n):
        raw = oracle.bits_to_word(arrs["raw_bits"][i])
        rec["raw"][i] = raw
        rec["status"][i] = arrs["has_corrected"][i]
        rec["msg"][i] = oracle.bits_to_word(arrs["corrected"][i]) if arrs["has_corrected"][i] else 0
        rec["errors"][i] = arrs["errors"][i]
        rec["matches"][i] = 60 - bin(raw ^ kcw).count("1")
        rec["verified"][i] = arrs["verified"][i]
    return rec


def test_records_json_matches_reference_dump(qrm, ref):
    # records from the reference itself, re-packed into the ABI record layout
    cfg = oracle.DetectCfg()
    code = qrm.resolve_profile("gf16-15-12")
    kcw = oracle.bits_to_word(oracle.Oracle().rs_encode(4, 15, 12, qrm.default_message(1, 48)))
    pos = list(ref.make_corpus(1000, 6, 256, 256, cfg))
    neg = list(ref.make_corpus(5000, 6, 256, 256, cfg, embed=False))
    imgs = pos + neg
    rec = _pack(qrm, ref.detect_batch(imgs, cfg)[0], kcw)
    got = qrm.records_json(rec, code)
    assert got == ref.detect_json(imgs, cfg)
    assert '"cache_hit": true' in got  # the watermarked images share one raw word
    assert qrm.records_json(rec, code, cache=(False, 4096, 1 << 20)) == ref.detect_json(imgs, cfg, cache=False)
    assert qrm.records_json(rec[:0], code) == "[]"
    # a tiny codebook exercises both eviction rules (staleness, then capacity)
    imgs2 = [pos[0], neg[0], neg[1], pos[1], neg[2], pos[2], neg[3], neg[4], neg[5], pos[3], pos[4], neg[0], pos[5]]
    rec2 = _pack(qrm, ref.detect_batch(imgs2, cfg)[0], kcw)
    for capy, stale in ((2, 1 << 20), (3, 2), (1, 1), (0, 5), (4096, 1 << 20)):
        assert qrm.records_json(rec2, code, cache=(True, capy, stale)) == \
            ref.detect_json(imgs2, cfg, cache_capacity=capy, stale_after=stale), (capy, stale)


@pytest.mark.gpu
def test_gpu_records_json_equals_reference_report(qrm, ref, cuda):
    """Images -> GPU detection -> JSON equals the reference pipeline's JSON byte for byte."""
    cfg = qrm.DetectionConfig()
    imgs = cuda.cat([qrm.make_corpus(cfg, 1000, 16), qrm.make_corpus(cfg, 5000, 16, embed=False)])
    host = imgs.cpu().numpy()
    with qrm.DetectionContext(cfg) as ctx:
        rec, _ = ctx.detect_host(host, 0)
    assert qrm.records_json(rec, cfg.code) == ref.detect_json(list(host), oracle.DetectCfg())
