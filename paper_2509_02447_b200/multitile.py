"""Multi-tile interleaving: per-image tile sizes placed on CUDA streams by
Algorithm 2 (BASELINE configs[2]; PAPER.md 6.2).

The reference defines the pieces but never runs them on real work:
``TileSizePredictor`` / ``ConstantTilePredictor`` (sched.hpp:73-86),
``WarmupStats`` with latency and memory scaling with tile area
(sched.cpp:126-136), ``build_tasks`` (sched.cpp:138-155) and ``lpt_schedule``
(sched.cpp:177-235). Here they drive the device path:

- the predictor picks each image's tile size;
- images of one size form a group, cut into mini-batch tasks whose latency and
  memory come from the warm-up statistics scaled by (tile / 64)^2;
- ``lpt_schedule`` (the C++ planner, bit-exact with the reference's) places and
  shards the tasks over S streams;
- one host thread per stream (a pool kept across calls) runs its pieces in placement order through the
  native executor (``qrm_detect_host_images``: only each image's window
  crosses PCIe). Each stream owns one context per tile size, because a
  context is single-size like the reference's (detect.hpp:114).

Tile sizes default to {32, 64, 128}: on 512^2 images the preprocess crops at
offset 128 and the cmd_bench corpus embeds its grid from (0, 0), so only sizes
dividing 128 keep detection tiles on the embedding grid (with 80 no watermark
verifies, in the reference as here).

Records of the images with tile size l equal one reference ``detect_batch``
over that size's sub-list in input order (draw index = position in the
sub-list), i.e. one single-size DetectionContext per size, as SURVEY 8(d)
row 3 describes.
"""
from __future__ import annotations

import dataclasses
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import RECORD_DTYPE, DetectionConfig, DetectionContext, InvalidInput, lpt_schedule


class TileSizePredictor:
    """sched.hpp:73-78: the tile-size oracle interface (the paper's learned predictor sits behind it)."""

    def select_tile_size(self, image: np.ndarray) -> int:
        raise NotImplementedError


class ConstantTilePredictor(TileSizePredictor):
    """sched.hpp:80-86."""

    def __init__(self, size: int):
        self.size = int(size)

    def select_tile_size(self, image: np.ndarray) -> int:
        return self.size


class ContrastTilePredictor(TileSizePredictor):
    """A deterministic stand-in for the learned predictor: the standard deviation
    of the green channel over the centre 256x256 crop. Low-contrast images get
    the larger tile (more pixels of evidence per bit), high-contrast images the
    smaller one."""

    def __init__(self, sizes=(128, 64, 32), thresholds=(46.0, 47.4)):
        self.sizes = tuple(int(s) for s in sizes)
        self.thresholds = tuple(float(t) for t in thresholds)

    def contrast(self, image: np.ndarray) -> float:
        h, w = image.shape[:2]
        y0, x0 = max(0, (h - 256) // 2), max(0, (w - 256) // 2)
        return float(image[y0:y0 + 256, x0:x0 + 256, 1].astype(np.float64).std())

    def select_tile_size(self, image: np.ndarray) -> int:
        c = self.contrast(image)
        if c < self.thresholds[0]:
            return self.sizes[0]
        if c < self.thresholds[1]:
            return self.sizes[1]
        return self.sizes[2]


@dataclass
class WarmupStats:
    """sched.cpp:126-136: latency and memory at a reference tile size, scaled by tile area."""
    reference_tile: int = 64
    detect_latency: float = 1.0  # ms per image at the reference tile
    detect_memory: float = 3 * 64 * 64  # bytes per image at the reference tile

    def latency_for(self, tile: int) -> float:
        r = tile / self.reference_tile
        return self.detect_latency * r * r

    def memory_for(self, tile: int) -> float:
        r = tile / self.reference_tile
        return self.detect_memory * r * r


def build_tasks(images, predictor: TileSizePredictor, stats: WarmupStats):
    """sched.cpp:138-155: one task per image -> [(id, tile, latency, memory)]."""
    if stats.reference_tile <= 0:
        raise InvalidInput("warm-up stats missing reference tile")
    tasks = []
    for i, img in enumerate(images):
        tile = int(predictor.select_tile_size(img))
        if tile <= 0:
            raise InvalidInput("predictor returned invalid tile size")
        lat = stats.latency_for(tile)
        if lat <= 0.0:
            raise InvalidInput("warm-up stats predict nonpositive latency")
        tasks.append((i, tile, lat, stats.memory_for(tile)))
    return tasks


def schedule_groups(counts, stats: WarmupStats, streams: int, minibatch: int, lam: float, b_min: int):
    """Algorithm 2 over per-size groups: each group of counts[l] images is cut into
    mini-batch tasks (latency / memory from the warm-up statistics), lpt_schedule
    places and shards them over `streams` streams, and each piece becomes a
    contiguous range (size, first, count) of its group. Returns (per-stream
    piece lists in placement order, stream loads)."""
    tasks = []
    for l in sorted(counts):
        for a in range(0, counts[l], minibatch):
            tasks.append((l, a, min(minibatch, counts[l] - a)))
    per_stream = [[] for _ in range(streams)]
    if not tasks:
        return per_stream, [0.0] * streams
    lat = [stats.latency_for(l) * c for (l, _, c) in tasks]
    mem = [stats.memory_for(l) * c for (l, _, c) in tasks]
    sch = lpt_schedule(list(range(len(tasks))), lat, mem, [c for (_, _, c) in tasks], streams, lam,
                       float(1 << 40), b_min, sum(counts.values()))
    offset = [0] * len(tasks)
    for (st, tid, units, _, _, _) in sch["pieces"]:
        l, a, _ = tasks[tid]
        per_stream[st].append((l, a + offset[tid], units))
        offset[tid] += units
    if offset != [c for (_, _, c) in tasks]:
        raise RuntimeError("schedule does not cover the batch")
    return per_stream, sch["loads"]


class MultiTileDetector:
    """Per-image tile sizes, Algorithm 2 placement over `streams` CUDA streams.

    ``detect(images)`` takes same-size host images (>= 256 px; a list of HxWx3
    uint8 arrays or one [N, H, W, 3] array) and returns records in input order
    plus the chosen sizes and the schedule."""

    def __init__(self, cfg: DetectionConfig, tile_sizes=(32, 64, 128), streams: int = 2, device: int = 0,
                 predictor: TileSizePredictor | None = None):
        if streams < 1:
            raise InvalidInput("need at least one stream")
        self.cfg = cfg
        self.tile_sizes = tuple(int(t) for t in tile_sizes)
        self.streams = int(streams)
        self.predictor = predictor or ContrastTilePredictor()
        self.ctx = [{l: DetectionContext(dataclasses.replace(cfg, tile_size=l), device=device)
                     for l in self.tile_sizes} for _ in range(self.streams)]
        self.stats = WarmupStats()
        self.pool = ThreadPoolExecutor(self.streams)  # one host thread per stream, kept across calls

    def close(self):
        self.pool.shutdown(wait=True)
        for per in self.ctx:
            for c in per.values():
                c.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def warmup(self, images, iters: int = 3, b0: int = 256) -> WarmupStats:
        """WarmupStats from the device path at the reference tile (64): median ms per
        image of b0-image batches, memory = window bytes per image."""
        imgs = list(images[:b0])
        ctx = self.ctx[0][64] if 64 in self.ctx[0] else next(iter(self.ctx[0].values()))
        ref = 64 if 64 in self.ctx[0] else self.tile_sizes[0]
        ts = []
        for _ in range(iters + 1):
            t0 = time.perf_counter()
            ctx.detect_images(imgs, 0)
            ts.append((time.perf_counter() - t0) * 1e3 / len(imgs))
        self.stats = WarmupStats(ref, float(np.median(ts[1:])), float(3 * ref * ref))
        return self.stats

    def detect(self, images, lam: float = 0.2, b_min: int = 128, minibatch: int = 512, sizes=None):
        imgs = [np.ascontiguousarray(im, dtype=np.uint8) for im in images]
        n = len(imgs)
        out = np.zeros(n, dtype=RECORD_DTYPE)
        if n == 0:
            return out, {"sizes": [], "pieces": []}
        if sizes is None:
            sizes = [t[1] for t in build_tasks(imgs, self.predictor, self.stats)]
        sizes = [int(s) for s in sizes]
        for s in set(sizes):
            if s not in self.tile_sizes:
                raise InvalidInput(f"predicted tile size {s} has no context")
        groups = {l: [i for i in range(n) if sizes[i] == l] for l in self.tile_sizes}
        per_stream, loads = schedule_groups({l: len(groups[l]) for l in self.tile_sizes}, self.stats, self.streams,
                                            minibatch, lam, b_min)
        errors = []

        def run(s):
            try:
                for (l, a, cnt) in per_stream[s]:
                    idx = groups[l][a:a + cnt]
                    rec, _ = self.ctx[s][l].detect_images([imgs[i] for i in idx], first_draw=a)
                    out[idx] = rec
            except Exception as exc:  # surfaced to the caller below
                errors.append(exc)

        for f in [self.pool.submit(run, s) for s in range(self.streams)]:
            f.result()
        if errors:
            raise errors[0]
        return out, {"sizes": sizes, "pieces": per_stream, "loads": loads,
                     "counts": {l: len(groups[l]) for l in self.tile_sizes}}

    def detect_grouped(self, groups, shape, lam: float = 0.2, b_min: int = 128, minibatch: int = 512):
        """The same schedule over images already grouped by tile size in page-locked
        host memory (an ingest stage that routes each image to its size's buffer):
        ``groups`` = {tile size: (host pointer, count)}, images of ``shape`` (H, W)
        back to back. Pieces are contiguous ranges, so each one takes the
        zero-copy window fetch (qrm_detect_host mode 0). Returns {size: records}."""
        H, W = shape
        img_bytes = H * W * 3
        counts = {l: int(groups[l][1]) if l in groups else 0 for l in self.tile_sizes}
        out = {l: np.zeros(counts[l], dtype=RECORD_DTYPE) for l in self.tile_sizes}
        if not any(counts.values()):
            return out, {"pieces": [], "counts": counts}
        per_stream, loads = schedule_groups(counts, self.stats, self.streams, minibatch, lam, b_min)
        errors = []

        def run(s):
            try:
                for (l, a, cnt) in per_stream[s]:
                    ptr = groups[l][0] + a * img_bytes
                    self.ctx[s][l].detect_host(None, a, plan=([1, 1, 1], [cnt] * 3), mode=0, out=out[l][a:a + cnt],
                                               ptr=ptr, shape=(cnt, H, W))
            except Exception as exc:
                errors.append(exc)

        for f in [self.pool.submit(run, s) for s in range(self.streams)]:
            f.result()
        if errors:
            raise errors[0]
        return out, {"pieces": per_stream, "loads": loads, "counts": counts}
