"""Multi-GPU sharding of the detection path.

Images are independent, so a batch shards into contiguous ranges, one per
rank (one process per GPU), with no collective on the data path. Each image
keeps its GLOBAL draw index (tiling.cpp:40 numbers tiles by position in the
list passed to detect_batch), so a sharded run reproduces one reference run
over the whole list. Records are gathered to the host of rank 0 only for
reporting (torch.distributed object gather over whatever backend the job
uses); no device-side exchange exists.
"""
from __future__ import annotations

import numpy as np


def shard_range(count: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) of rank `rank`; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(count, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def merge_records(parts: list[tuple[int, np.ndarray]], count: int) -> np.ndarray:
    """Concatenate per-rank record arrays (begin, records) in image order."""
    parts = sorted(parts, key=lambda p: p[0])
    out = np.concatenate([p[1] for p in parts]) if parts else np.zeros(0)
    if out.shape[0] != count:
        raise ValueError(f"gathered {out.shape[0]} records for {count} images")
    pos = 0
    for begin, recs in parts:
        if begin != pos:
            raise ValueError("shards are not contiguous")
        pos += recs.shape[0]
    return out


def detect_sharded(images, cfg, detect_fn, dist=None):
    """Run `detect_fn(shard_images, first_draw)` on this rank's shard and
    gather all shards' records on rank 0 (None elsewhere).

    `detect_fn` is the per-rank decoder (e.g. DetectionContext.detect_host on
    the rank's GPU); the draw index passed is the shard's global offset."""
    world = dist.get_world_size() if dist is not None else 1
    rank = dist.get_rank() if dist is not None else 0
    count = len(images)
    b, e = shard_range(count, world, rank)
    recs = detect_fn(images[b:e], b)
    if dist is None:
        return merge_records([(b, recs)], count)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((b, recs), gathered, dst=0)
    return merge_records(gathered, count) if rank == 0 else None
