"""Host-side multi-rank logic on CPU (gloo, world_size 2): contiguous shards,
global draw indices and the record gather reproduce a single run over the
whole batch. The per-rank decoder here is the C oracle (CPU), standing in for
each rank's GPU; the sharding/merge code under test is the product's."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_02447_b200.shard import detect_sharded, merge_records, shard_range


def test_shard_ranges_cover_exactly():
    for count in (0, 1, 7, 64, 1000003):
        for world in (1, 2, 3, 8):
            rs = [shard_range(count, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == count
            for (a, b), (c, d) in zip(rs, rs[1:]):
                assert b == c
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_merge_rejects_gaps():
    a = np.zeros(3)
    with pytest.raises(ValueError):
        merge_records([(0, a), (4, a)], 7)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    o = oracle.Oracle()
    cfg = oracle.DetectCfg()
    images = np.concatenate([o.make_corpus(1000, 10, 256, 256, cfg), o.make_corpus(5000, 10, 256, 256, cfg, embed=False)])

    def decode(shard, first_draw):
        r = o.detect(list(shard), cfg, first_draw=first_draw)
        return np.stack([r["raw"], r["msg"], r["decoded"].astype(np.uint64), r["verified"].astype(np.uint64)], 1)

    merged = detect_sharded(images, cfg, decode, dist)
    if rank == 0:
        np.save(out_path, merged)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_matches_single_run(tmp_path):
    import oracle
    out = str(tmp_path / "merged.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    merged = np.load(out)
    o = oracle.Oracle()
    cfg = oracle.DetectCfg()
    images = np.concatenate([o.make_corpus(1000, 10, 256, 256, cfg), o.make_corpus(5000, 10, 256, 256, cfg, embed=False)])
    r = o.detect(list(images), cfg, first_draw=0)
    single = np.stack([r["raw"], r["msg"], r["decoded"].astype(np.uint64), r["verified"].astype(np.uint64)], 1)
    assert np.array_equal(merged, single)
    assert merged[:10, 3].all() and not merged[10:, 3].any()
