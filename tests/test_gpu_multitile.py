"""Multi-tile interleaving (BASELINE configs[2]): per-image tile sizes {32, 64, 128}
placed on two CUDA streams by Algorithm 2, records equal one single-size run per
size and the compiled reference on each size's sub-list."""
import dataclasses

import numpy as np
import pytest

from test_gpu_detect import _ocfg, assert_records_equal, ref_fields

pytestmark = pytest.mark.gpu


def _mixed_corpus(qrm, cfg, n, sizes_cycle=(32, 64, 128)):
    """512^2 images, image i embedded with tile size sizes_cycle[i % 3] (so the
    size it will be detected with); every 5th image unwatermarked."""
    sizes = [sizes_cycle[i % len(sizes_cycle)] for i in range(n)]
    imgs = [None] * n
    for l in sizes_cycle:
        idx = [i for i in range(n) if sizes[i] == l]
        cl = dataclasses.replace(cfg, tile_size=l)
        pos = qrm.make_corpus(cl, 7000 + l, len(idx), 512, 512).cpu().numpy()
        neg = qrm.make_corpus(cl, 9000 + l, len(idx), 512, 512, embed=False).cpu().numpy()
        for j, i in enumerate(idx):
            imgs[i] = neg[j] if i % 5 == 4 else pos[j]
    return imgs, sizes


def test_multitile_lpt_equals_single_size_runs_and_reference(qrm, cuda, ref):
    from paper_2509_02447_b200.multitile import MultiTileDetector
    cfg = qrm.DetectionConfig()
    imgs, sizes = _mixed_corpus(qrm, cfg, 150)
    with MultiTileDetector(cfg, streams=2) as mt:
        mt.warmup(imgs, iters=1, b0=32)
        got, info = mt.detect(imgs, sizes=sizes, minibatch=16, b_min=4, lam=0.2)
        assert sum(len(p) for p in info["pieces"]) >= 2 and all(info["pieces"])  # both streams worked
        for l in (32, 64, 128):
            idx = [i for i in range(len(imgs)) if sizes[i] == l]
            cl = dataclasses.replace(cfg, tile_size=l)
            with qrm.DetectionContext(cl) as ctx:
                one, _ = ctx.detect_images([imgs[i] for i in idx], 0)
            assert np.array_equal(got[idx], one)
            want = ref_fields(ref.detect_sequential([imgs[i] for i in idx], _ocfg(cl), first_draw=0, cache=False),
                              cl.code)
            assert_records_equal(qrm.semantic_fields(got[idx], cl.code), want)
            emb = [j for j, i in enumerate(idx) if i % 5 != 4]
            rate = got[idx]["verified"][emb].mean()
            print(f"tile {l}: verified {rate:.2f} of watermarked")
            if l >= 64:  # 32x32 tiles carry a quarter of the evidence: at alpha 0.04 most fail RS (as in the reference)
                assert rate > 0.9


def test_multitile_grouped_pinned_equals_list_path(qrm, cuda):
    """detect_grouped (per-size page-locked buffers, zero-copy window fetch) gives
    the list path's records."""
    from paper_2509_02447_b200.multitile import MultiTileDetector
    cfg = qrm.DetectionConfig()
    imgs, sizes = _mixed_corpus(qrm, cfg, 90)
    with MultiTileDetector(cfg, streams=2) as mt:
        ref_recs, _ = mt.detect(imgs, sizes=sizes, minibatch=8, b_min=4)
        groups, keep = {}, []
        for l in (32, 64, 128):
            idx = [i for i in range(len(imgs)) if sizes[i] == l]
            buf = cuda.empty((len(idx), 512, 512, 3), dtype=cuda.uint8, pin_memory=True)
            buf.copy_(cuda.from_numpy(np.stack([imgs[i] for i in idx])))
            keep.append(buf)
            groups[l] = (buf.data_ptr(), len(idx))
        got, info = mt.detect_grouped(groups, (512, 512), minibatch=8, b_min=4)
        for l in (32, 64, 128):
            idx = [i for i in range(len(imgs)) if sizes[i] == l]
            assert np.array_equal(got[l], ref_recs[idx])


def test_multitile_predictor_path(qrm, cuda):
    """Sizes from the ContrastTilePredictor (build_tasks) instead of given sizes."""
    from paper_2509_02447_b200.multitile import ContrastTilePredictor, MultiTileDetector, build_tasks
    cfg = qrm.DetectionConfig()
    imgs, _ = _mixed_corpus(qrm, cfg, 60)
    with MultiTileDetector(cfg, streams=3) as mt:
        got, info = mt.detect(imgs, minibatch=8, b_min=2)
    pred = [t[1] for t in build_tasks(imgs, ContrastTilePredictor(), mt.stats)]
    assert info["sizes"] == pred and got.shape[0] == 60
