"""The C oracle against the golden vectors produced by the compiled reference
(tests/golden/make_golden.py) and the reference's own test expectations
(proj/tests/test_gf.cpp, test_rs.cpp, test_image.cpp). CPU only."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def kat():
    with open(os.path.join(G, "kat.json")) as f:
        return json.load(f)


def test_key_message_and_codewords(orc, kat):
    msg = orc.default_message(1, 48)
    assert format(oracle.bits_to_word(msg), "012x") == kat["default_message_hex"] == "b1b8528ad785"
    assert format(oracle.bits_to_word(orc.rs_encode(4, 15, 12, msg)), "015x") == kat["gf16_codeword_hex"]
    assert kat["gf16_codeword_hex"] == "b1b8528ad7859a0"
    assert format(oracle.bits_to_word(orc.rs_encode(8, 8, 6, msg)), "016x") == kat["gf256_codeword_hex"]


def test_verify_thresholds(orc, kat):
    for n, tau in kat["tau_1e-6"].items():
        assert orc.verify_threshold(int(n), 1e-6) == tau
    for n, f, tau in kat["tau_misc"]:
        assert orc.verify_threshold(n, f) == tau
    assert kat["tau_1e-6"]["48"] == 41 and kat["tau_1e-6"]["60"] == 49 and kat["tau_1e-6"]["64"] == 51


def test_rng_words(orc, kat):
    for s, st, c, v in kat["rng_word"]:
        assert orc.rng_word(s, st, c) == int(v)


def test_select_tile(orc, kat):
    for w, h, l, strat, seed, draw, x, y in kat["select_tile"]:
        assert orc.select_tile(w, h, l, strat, seed, draw) == (x, y)


@pytest.mark.parametrize("name,mnk", [("gf16", (4, 15, 12)), ("gf256", (8, 8, 6))])
def test_rs_vectors(orc, name, mnk):
    d = np.load(os.path.join(G, f"rs_{name}.npz"))
    cw, ne = orc.bw_decode_packed(*mnk, d["words"])
    assert np.array_equal(ne, d["nerr"])
    assert np.array_equal(cw[ne >= 0], d["cw"][ne >= 0])
    assert (ne == -1).sum() > 100 and (ne == 1).sum() > 100  # both outcomes exercised


def test_gf_tables_against_clmul(orc):
    """test_gf.cpp:17-22, 48-60: table multiply == carry-less multiply mod poly."""
    def clmul(a, b, poly, m):
        acc = 0
        for i in range(m):
            if (b >> i) & 1:
                acc ^= a << i
        for d in range(2 * m - 2, m - 1, -1):
            if (acc >> d) & 1:
                acc ^= poly << (d - m)
        return acc
    for a in range(16):
        for b in range(16):
            assert orc.lib.orc_gf_mul(4, a, b) == clmul(a, b, 0x13, 4)
    rng = np.random.default_rng(3)
    for a, b in rng.integers(0, 256, size=(2000, 2)):
        assert orc.lib.orc_gf_mul(8, int(a), int(b)) == clmul(int(a), int(b), 0x11D, 8)


def test_rs_reference_test_cases(orc):
    """test_rs.cpp:60-163 expectations on the oracle."""
    assert not orc.rs_encode(4, 15, 12, np.zeros(48, np.uint8)).any()
    rng = np.random.default_rng(22)
    for _ in range(50):
        msg = rng.integers(0, 2, 48).astype(np.uint8)
        cw = orc.rs_encode(4, 15, 12, msg)
        assert np.array_equal(cw[:48], msg)
        res = orc.bw_decode(4, 15, 12, cw)
        assert res is not None and res[2] == 0 and np.array_equal(res[0], msg)
    # exhaustive single-symbol corruption for 3 messages
    for _ in range(3):
        msg = rng.integers(0, 2, 48).astype(np.uint8)
        cw = oracle.bits_to_word(orc.rs_encode(4, 15, 12, msg))
        for pos in range(15):
            for v in range(1, 16):
                bad = cw ^ (v << (4 * (14 - pos)))
                res = orc.bw_decode(4, 15, 12, oracle.word_to_bits(bad, 60))
                assert res is not None and res[2] == 1 and np.array_equal(res[0], msg)
    # t=2 (12,8) double errors
    for _ in range(40):
        msg = rng.integers(0, 2, 64).astype(np.uint8)
        cwb = orc.rs_encode(8, 12, 8, msg)
        sym = [oracle.bits_to_word(cwb[8 * j:8 * j + 8]) for j in range(12)]
        p1, p2 = rng.choice(12, 2, replace=False)
        sym[p1] ^= int(rng.integers(1, 256))
        sym[p2] ^= int(rng.integers(1, 256))
        bits = np.concatenate([oracle.word_to_bits(s, 8) for s in sym])
        res = orc.bw_decode(8, 12, 8, bits)
        assert res is not None and res[2] == 2 and np.array_equal(res[0], msg)


def test_detect_records(orc):
    d = np.load(os.path.join(G, "detect_256.npz"))
    cfg = oracle.DetectCfg()
    imgs = np.concatenate([orc.make_corpus(1000, 24, 256, 256, cfg), orc.make_corpus(5000, 24, 256, 256, cfg,
                                                                                        embed=False)])
    assert hashlib.sha256(imgs.tobytes()).hexdigest() == str(d["corpus_sha256"])
    O = orc.detect(list(imgs), cfg)
    raw = np.array([oracle.bits_to_word(b) for b in d["raw_bits"]], np.uint64)
    assert np.array_equal(O["raw"], raw)
    assert np.array_equal(O["decoded"].astype(bool), d["has_corrected"].astype(bool))
    msg = np.array([oracle.bits_to_word(b) if h else 0 for b, h in zip(d["corrected"], d["has_corrected"])],
                   np.uint64)
    assert np.array_equal(np.where(O["decoded"] == 1, O["msg"], 0).astype(np.uint64), msg)
    assert np.array_equal(O["errors"], d["errors"])
    assert np.array_equal(O["bit_acc"], d["bit_acc"])
    assert np.array_equal(O["verified"].astype(bool), d["verified"].astype(bool))
    assert d["verified"][:24].all() and not d["verified"][24:].any()


def test_extract_soft(orc):
    soft = np.load(os.path.join(G, "extract_soft.npy"))
    cfg = oracle.DetectCfg()
    imgs = orc.make_corpus(1000, 6, 256, 256, cfg)
    for i in range(6):
        x, y = orc.select_tile(256, 256, 64, "random_grid", 0, i)
        tile = (imgs[i, y:y + 64, x:x + 64].astype(np.float64) / 127.5 - 1.0).astype(np.float32)
        assert np.array_equal(orc.extract(1, 60, 64, tile), soft[i])  # same summation order: bit-identical


def test_preprocess(orc):
    d = np.load(os.path.join(G, "preprocess.npz"))
    for (w, h) in [(1, 1), (300, 200), (100, 300), (255, 255), (512, 384)]:
        out = orc.preprocess(orc.synthetic_image(w * 31 + h, w, h))
        assert hashlib.sha256(out.tobytes()).hexdigest() == str(d[f"{w}x{h}_sha256"])
        assert np.array_equal(out.reshape(-1)[::97], d[f"{w}x{h}_sample"])


def test_schedulers(orc, kat):
    for c in kat["allocate_streams"]:
        rc, s, mb, bn = orc.allocate_streams(c["time"], c["memory"], c["b0"], c["B"], c["P"], c["m_cap"], c["eps"],
                                             c["stall"])
        assert rc == c["rc"]
        if rc == 0:
            assert (s, mb, bn) == (c["streams"], c["minibatch"], c["bottleneck"])
    for c in kat["lpt_schedule"]:
        lam = float("inf") if c["lam"] == "inf" else c["lam"]
        rc, out = orc.lpt_schedule(c["ids"], c["lat"], c["mem"], c["units"], c["S"], lam, c["m_cap"], c["b_min"],
                                   c["B"])
        assert rc == c["rc"]
        if rc == 0:
            assert [list(p) for p in out["pieces"]] == [list(p) for p in c["out"]["pieces"]]
            assert out["loads"] == c["out"]["loads"] and out["m_unit"] == c["out"]["m_unit"]
