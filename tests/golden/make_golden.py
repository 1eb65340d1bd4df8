"""Generate the golden fixtures in tests/golden/ from the COMPILED REFERENCE.

Run in a container that has /root/reference (it builds oracle/_ref from the
reference sources in place):  python tests/golden/make_golden.py

Every value below comes from the reference library's own public API through
oracle/ref_harness.cpp; the fixtures pin the C oracle (tests/test_oracle_golden.py)
on hosts where the reference itself is absent (the GPU box).
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main():
    r = oracle.Reference()
    kat = {}
    msg = r.default_message(1, 48)
    kat["default_message_hex"] = format(oracle.bits_to_word(msg), "012x")
    kat["gf16_codeword_hex"] = format(oracle.bits_to_word(r.rs_encode(4, 15, 12, msg)), "015x")
    kat["gf256_codeword_hex"] = format(oracle.bits_to_word(r.rs_encode(8, 8, 6, msg)), "016x")
    kat["tau_1e-6"] = {str(n): r.verify_threshold(n, 1e-6) for n in list(range(1, 101)) + [128, 200]}
    kat["tau_misc"] = [[n, f, r.verify_threshold(n, f)] for n in (16, 48, 60, 64, 96)
                       for f in (0.5, 1e-2, 1e-4, 1e-9, 2.0 ** -48)]
    kat["rng_word"] = [[s, st, c, str(r.rng_word(s, st, c))] for s in (0, 1, 2 ** 63 + 5)
                       for st in (0, 7, 0x6D73) for c in (0, 1, 12287, 2 ** 40 + 3)]
    rng = np.random.default_rng(11)
    tiles = []
    for _ in range(300):
        w, h = int(rng.integers(64, 700)), int(rng.integers(64, 700))
        l = int(rng.choice([16, 32, 64, 80]))
        if l > min(w, h):
            continue
        strat = ["random", "random_grid", "fixed"][int(rng.integers(0, 3))]
        seed, draw = int(rng.integers(0, 2 ** 62)), int(rng.integers(0, 2 ** 40))
        tiles.append([w, h, l, strat, seed, draw, *r.select_tile(w, h, l, strat, seed, draw)])
    kat["select_tile"] = tiles

    # allocate_streams / lpt_schedule cases (SPEC.md:484-520 shapes)
    sched = []
    for case in range(40):
        K = int(rng.integers(2, 5))
        t = rng.uniform(0.5, 30, size=K).round(3).tolist()
        u = rng.uniform(0, 1e6, size=K).round(1).tolist()
        B = int(rng.integers(1, 600))
        P = int(rng.integers(K, 24))
        cap = float(rng.choice([1e7, 1e9, 5e10]))
        eps = float(rng.choice([0.0, 0.01, 0.5]))
        stall = int(rng.integers(1, 4))
        rc, s, mb, bn = r.allocate_streams(t, u, 16, B, P, cap, eps, stall)
        sched.append({"time": t, "memory": u, "b0": 16, "B": B, "P": P, "m_cap": cap, "eps": eps, "stall": stall,
                      "rc": rc, "streams": s, "minibatch": mb, "bottleneck": bn})
    kat["allocate_streams"] = sched
    lpt = []
    for case in range(40):
        n = int(rng.integers(1, 14))
        ids = list(range(n))
        lat = rng.uniform(0.1, 9, size=n).round(2).tolist()
        mem = rng.uniform(0, 50, size=n).round(1).tolist()
        units = rng.integers(1, 9, size=n).tolist()
        S = int(rng.integers(1, 5))
        lam = float(rng.choice([0.0, 0.1, 0.5, float("inf")]))
        cap = float(rng.choice([1e9, 200.0]))
        b_min = int(rng.integers(1, 4))
        B = int(rng.integers(1, 200))
        rc, out = r.lpt_schedule(ids, lat, mem, units, S, lam, cap, b_min, B)
        lpt.append({"ids": ids, "lat": lat, "mem": mem, "units": units, "S": S, "lam": "inf" if lam == float("inf")
                    else lam, "m_cap": cap, "b_min": b_min, "B": B, "rc": rc, "out": out})
    kat["lpt_schedule"] = lpt
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=0)

    # RS vectors: packed gf16 / gf256-dynamic(48), mixed error counts + random words
    for name, (m, n, k) in {"gf16": (4, 15, 12), "gf256": (8, 8, 6)}.items():
        N = 4000
        words = []
        for i in range(N):
            mb = rng.integers(0, 2, size=k * m).astype(np.uint8)
            cw = oracle.bits_to_word(r.rs_encode(m, n, k, mb))
            e = int(rng.integers(0, 4))
            for p in rng.choice(n, size=e, replace=False):
                cw ^= int(rng.integers(1, 1 << m)) << (m * (n - 1 - int(p)))
            words.append(cw)
        words += [int(x) for x in rng.integers(0, 2 ** 62, size=1000)]
        words = np.array(words, dtype=np.uint64) & np.uint64((1 << (n * m)) - 1)
        cw, ne, _ = r.bw_decode_packed(m, n, k, words)
        np.savez_compressed(os.path.join(HERE, f"rs_{name}.npz"), words=words, cw=cw, nerr=ne)

    # Detection records on the cmd_bench corpus (embedded + negatives) and 512^2 / odd sizes
    cfg = oracle.DetectCfg()
    pos = r.make_corpus(1000, 24, 256, 256, cfg)
    neg = r.make_corpus(5000, 24, 256, 256, cfg, embed=False)
    imgs = np.concatenate([pos, neg])
    R = r.detect_sequential(list(imgs), cfg)
    np.savez_compressed(os.path.join(HERE, "detect_256.npz"), raw_bits=R["raw_bits"], corrected=R["corrected"],
                        has_corrected=R["has_corrected"], errors=R["errors"], bit_acc=R["bit_acc"],
                        verified=R["verified"], corpus_sha256=hashlib.sha256(imgs.tobytes()).hexdigest())
    # extract soft values for 6 tiles
    soft = []
    for i in range(6):
        x, y = r.select_tile(256, 256, 64, "random_grid", 0, i)
        tile = (imgs[i, y:y + 64, x:x + 64].astype(np.float64) / 127.5 - 1.0).astype(np.float32)
        soft.append(r.extract(1, 60, 0.04, 64, tile))
    np.save(os.path.join(HERE, "extract_soft.npy"), np.array(soft))
    # preprocess of odd sizes
    pre = {}
    for (w, h) in [(1, 1), (300, 200), (100, 300), (255, 255), (512, 384)]:
        img = r.synthetic_image(w * 31 + h, w, h)
        out = r.preprocess(img)
        pre[f"{w}x{h}_sha256"] = np.array(hashlib.sha256(out.tobytes()).hexdigest())
        pre[f"{w}x{h}_sample"] = out.reshape(-1)[::97].copy()
    np.savez_compressed(os.path.join(HERE, "preprocess.npz"), **pre)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
