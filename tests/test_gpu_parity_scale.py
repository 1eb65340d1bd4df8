"""Parity at the exact bench geometries (BASELINE configs[1], [2], [4]).

Every record of a full bench-size batch is diffed against the compiled
reference (oracle/_ref: the unmodified detect pipeline) with the reference's
semantic_equal fields (detect.cpp:25-29). At these sizes the decode kernel
runs its production launch shapes (split-K clusters, 125-image tiles, 132+
CTAs, several waves), which the small-batch tests never reach. The reference
side runs in parallel chunks (detect_sequential with the chunk's global draw
offset; the ctypes calls release the GIL).

Learned extractor: 64 randomly sampled tiles of a full 4096-tile persistent-
kernel batch against the fp32 oracle (oracle/hidden_oracle.c), under the
tolerance of tests/test_hidden.py.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from test_gpu_detect import _ocfg, assert_records_equal, ref_fields

pytestmark = pytest.mark.gpu

THREADS = 16


def ref_records(ref, images, cfg, first_draw=0, chunk=256):
    """Reference records of `images` (uint8 [N, H, W, 3]) with draw index first_draw + i."""
    n = images.shape[0]
    oc = _ocfg(cfg)

    def run(b):
        e = min(n, b + chunk)
        return ref.detect_sequential(list(images[b:e]), oc, first_draw=first_draw + b, cache=False)

    with ThreadPoolExecutor(THREADS) as ex:
        parts = list(ex.map(run, range(0, n, chunk)))
    return {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}


def _mixed_256(qrm, cuda, cfg, n):
    """n/4 clean watermarked, n/4 blurred watermarked (bit errors -> RS corrections),
    n/2 unwatermarked (decode failures, exact-zero correlations)."""
    q = n // 4
    pos = qrm.make_corpus(cfg, 1000, 2 * q)
    blurred = qrm.apply_attack(pos[q:], "blur", 1.0)
    neg = qrm.make_corpus(cfg, 50000, n - 2 * q, embed=False)
    return cuda.cat([pos[:q], blurred, neg]).contiguous()


def _summary(rec):
    return {"decoded": int((rec["status"] == 1).sum()), "corrected": int(((rec["status"] == 1) & (rec["errors"] > 0)).sum()),
            "failed": int((rec["status"] == 0).sum()), "ties": int((rec["ties"] > 0).sum()),
            "verified": int(rec["verified"].sum())}


def test_configs1_batch4096_every_record(qrm, cuda, ref):
    """configs[1]: one 4096-image 256^2 batch through the three production entry
    points (device-resident decode, host executor mode 0, the drop-in's per-image
    staged path), every record against the reference."""
    cfg = qrm.DetectionConfig()
    imgs = _mixed_256(qrm, cuda, cfg, 4096)
    host = imgs.cpu().numpy()
    want = ref_fields(ref_records(ref, host, cfg, first_draw=8192), cfg.code)
    with qrm.DetectionContext(cfg) as ctx:
        dev = qrm.records_from_device(ctx.detect_device(imgs, first_draw=8192))
        hst, _ = ctx.detect_host(host, 8192)
        per, info = ctx.detect_images(list(host), 8192)
    for got in (dev, hst, per):
        assert_records_equal(qrm.semantic_fields(got, cfg.code), want)
    s = _summary(dev)
    print("configs[1] 4096:", s)
    # the batch exercises every record path: clean, corrected, failed, tied
    assert s["corrected"] > 0 and s["failed"] > 0 and s["ties"] > 0 and s["verified"] >= 2048
    assert min(info["busy_ns"]) > 0


def test_configs2_batch16384_512px_every_record(qrm, cuda, ref):
    """configs[2]: one 16,384-image 512^2 batch (12.9 GB on the device; centre crop
    at offset 128 keeps the tiles grid-aligned with the embedding), half
    watermarked; plus a 2048-image slice of it through the host executor."""
    cfg = qrm.DetectionConfig()
    n = 16384
    imgs = cuda.empty((n, 512, 512, 3), dtype=cuda.uint8, device="cuda")
    qrm.make_corpus(cfg, 7000, n // 2, 512, 512, out=imgs[: n // 2])
    qrm.make_corpus(cfg, 90000, n // 2, 512, 512, embed=False, out=imgs[n // 2:])
    with qrm.DetectionContext(cfg) as ctx:
        dev = qrm.records_from_device(ctx.detect_device(imgs, first_draw=0))
        cuda.cuda.synchronize()
        step = 2048
        for b in range(0, n, step):  # the reference in host-memory-sized pieces
            host = imgs[b:b + step].cpu().numpy()
            want = ref_fields(ref_records(ref, host, cfg, first_draw=b), cfg.code)
            assert_records_equal(qrm.semantic_fields(dev[b:b + step], cfg.code), want)
            if b in (0, n // 2):
                got, _ = ctx.detect_host(host, b, plan=([1, 2, 1], [1024] * 3))
                assert np.array_equal(got, dev[b:b + step])
    s = _summary(dev)
    print("configs[2] 16384 x 512^2:", s)
    assert s["verified"] >= n // 2 and s["failed"] > 0


def test_configs4_slice65536_host_pipeline(qrm, cuda, ref):
    """configs[4]: a 65,536-image slice of the 1M-image job exactly as bench.py
    runs it -- 4096-image calls of qrm_detect_host (mode 0, the default plan)
    cycling over a 16,384-image pinned pool, global draw index per image."""
    cfg = qrm.DetectionConfig()
    pool_n, call = 16384, 4096
    dev_pool = cuda.cat([qrm.make_corpus(cfg, 1000, pool_n // 2), qrm.make_corpus(cfg, 70000, pool_n // 2, embed=False)])
    pinned = cuda.empty(dev_pool.shape, dtype=cuda.uint8, pin_memory=True)
    pinned.copy_(dev_pool)
    host = pinned.numpy()
    del dev_pool
    total = 65536
    with qrm.DetectionContext(cfg) as ctx:
        for first in range(0, total, call):
            off = first % pool_n
            got, _ = ctx.detect_host(ptr=pinned[off:off + call].data_ptr(), shape=(call, 256, 256), first_draw=first)
            want = ref_fields(ref_records(ref, host[off:off + call], cfg, first_draw=first), cfg.code)
            assert_records_equal(qrm.semantic_fields(got, cfg.code), want)


def test_conv_extractor_sampled_tiles_of_4096_batch(qrm, cuda, orc):
    """Learned extractor at the bench geometry (4096 tiles, persistent kernels over
    all SMs): 64 randomly sampled tiles against the fp32 oracle."""
    from test_hidden import NB, NEAR_ZERO, REL_L2_TOL, SEED
    cfg = qrm.DetectionConfig()
    imgs = cuda.cat([qrm.make_corpus(cfg, 1000, 2048), qrm.make_corpus(cfg, 40000, 2048, embed=False)])
    with qrm.DetectionContext(cfg) as ctx:
        lg, rec = ctx.hidden_detect_device(imgs, weight_seed=SEED, first_draw=4096)
        cuda.cuda.synchronize()
    lg = lg.cpu().numpy().astype(np.float64)
    rec = qrm.records_from_device(rec)
    idx = np.sort(np.random.default_rng(2509).choice(4096, 64, replace=False))
    host = imgs[idx].cpu().numpy()

    def one(j):
        x, y = orc.select_tile(256, 256, 64, "random_grid", 0, 4096 + int(idx[j]))
        return orc.hidden_forward(SEED, NB, np.ascontiguousarray(host[j, y:y + 64, x:x + 64]))[0]

    with ThreadPoolExecutor(THREADS) as ex:
        want = np.array(list(ex.map(one, range(len(idx)))))
    got = lg[idx]
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    print(f"64 sampled tiles of 4096: logit rel L2 = {rel:.3e}")
    assert rel <= REL_L2_TOL
    confident = np.abs(want) > NEAR_ZERO * np.sqrt(np.mean(want ** 2))
    assert np.array_equal((got > 0)[confident], (want > 0)[confident])
    gpu_bits = np.array([oracle.bits_to_word((row > 0).astype(np.uint8)) for row in got], np.uint64)
    assert np.array_equal(rec["raw"][idx], gpu_bits)
