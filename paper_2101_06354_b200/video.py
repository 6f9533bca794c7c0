"""Frame-sequence driver: pinned-host staging, async H2D, batched scoring.

This is the B200 counterpart of the reference's frame loop
(``run_score``, src/pipeline.py:275-366, optional ThreadPoolExecutor at
:319-322) for the luma / multiscale / channel-wise color models: frames are
packed into a pinned host ring (two slots), uploaded on a dedicated copy
stream while the previous batch is being scored on the compute stream, and
only per-frame scalars come back.  Results are in frame order, one record per
frame with the pipeline's fields (score, am, l_mean, cs_mean;
src/pipeline.py:57-58, :230-236), then pooled over time with the configured
temporal pooler (src/pooling.py:246-280).

Multi-GPU: ``shard_bounds`` splits frame indices into contiguous per-rank
blocks (every frame pair is independent, so no collective is on the data
path); ``gather_frame_scores`` concatenates the per-rank score vectors after
scoring, in frame order.
"""

from __future__ import annotations

import os
import warnings
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _native as nat
from . import batch as B
from .errors import EmptySeries, ValidationError
from .options import SsimConfig
from .planes import ScoreSeries
from .pipeline import FrameScore, luma_records, score_frame_pair  # noqa: F401  (re-exported)
from .pooling import pool_temporal


@dataclass
class FrameRecord:
    frame: int
    score: float
    am: Optional[float]
    l_mean: Optional[float]
    cs_mean: Optional[float]


@dataclass
class SequenceResult:
    records: list = field(default_factory=list)
    pooled: float = float("nan")
    h2d_bytes: int = 0

    @property
    def scores(self) -> np.ndarray:
        return np.array([r.score for r in self.records], dtype=np.float64)


def shard_bounds(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [start, stop) of frame indices owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValidationError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_frame_scores(local: np.ndarray, n_frames: int, group=None) -> np.ndarray:
    """All ranks' per-frame scores concatenated in frame order (after scoring; off the hot path)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = [shard_bounds(n_frames, r, world) for r in range(world)]
    width = max(stop - start for start, stop in counts)
    buf = torch.full((width,), float("nan"), dtype=torch.float64)
    buf[: local.size] = torch.from_numpy(np.asarray(local, dtype=np.float64))
    if dist.get_backend(group) == "nccl":
        buf = buf.cuda()
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = [p.cpu().numpy()[: stop - start] for p, (start, stop) in zip(parts, counts)]
    return np.concatenate(out)


def _copy_into(job) -> None:
    dst, src = job
    np.copyto(dst, src, casting="unsafe")


class SequenceScorer:
    """Score a stream of frame pairs on one GPU.

    ``color_weights`` (3-tuple) scores YCbCr frames given as (Y, Cb, Cr) plane
    tuples with ``fixed_weight_cssim``; otherwise frames are luma planes.
    ``config.multiscale`` enabled -> MS-SSIM per frame (score only, as in the
    reference pipeline, src/pipeline.py:224-226).
    """

    def __init__(self, config: SsimConfig = SsimConfig(), batch_frames: int = 16,
                 color_weights: Optional[Sequence[float]] = None, device=None):
        self.config = config
        self.batch_frames = max(1, int(batch_frames))
        self.color_weights = tuple(color_weights) if color_weights is not None else None
        self.device = device or nat.require_device()
        torch = nat.torch_mod()
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self._slots = [None, None]
        self._copier = ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1))
        self._events = [None, None]   # upload of the slot finished (host buffer reusable)
        self._done = [None, None]     # scoring of the slot finished (device buffer reusable)

    # -- staging ------------------------------------------------------------
    def _stage(self, slot: int, frames: list, direct: bool = False):
        """Pack a batch into pinned slot memory and upload it on the copy stream.

        ``direct``: the frame planes already live in page-locked host memory (a pinned
        ``FrameSource``); planes whose rows need no padding are then DMA'd straight into
        the device slot, without the host packing copy."""
        torch = nat.torch_mod()
        nplanes = 3 if self.color_weights is not None else 1
        planes_ref, planes_dist = [], []
        shapes = []
        for p in range(nplanes):
            r0 = np.asarray(frames[0][0][p] if nplanes == 3 else frames[0][0])
            shapes.append((r0.shape, r0.dtype))
        # slot buffers hold batch_frames frames and are reused for shorter (final) batches:
        # pinned allocations are expensive, so they happen once per geometry
        key = (tuple(s for s, _ in shapes), tuple(str(d) for _, d in shapes))
        slot_bufs = self._slots[slot]
        if slot_bufs is None or slot_bufs[0] != key:
            bufs = []
            for (h, w), dt in shapes:
                t_dt = torch.uint8 if dt == np.uint8 else torch.uint16
                pitch = nat.aligned_pitch(w, nat.U8 if dt == np.uint8 else nat.U16)
                host = torch.empty((2, self.batch_frames, h, pitch), dtype=t_dt, pin_memory=True)
                dev = torch.empty_like(host, device=self.device)
                bufs.append((host, dev, w))
            slot_bufs = (key, bufs)
            self._slots[slot] = slot_bufs
        nf = len(frames)
        slot_bufs = (slot_bufs[0], [(host[:, :nf], dev[:, :nf], w) for host, dev, w in slot_bufs[1]])
        if self._events[slot] is not None:
            self._events[slot].synchronize()  # host slot free again (its upload finished)
        nbytes = 0
        with torch.cuda.stream(self.copy_stream):
            if self._done[slot] is not None:
                self.copy_stream.wait_event(self._done[slot])
            # pack all planes of the batch into the pinned slot with a thread pool (numpy
            # copies release the GIL, so the host memcpy runs on several cores), then
            # issue one async H2D per plane
            jobs = []
            dma = []
            for p, (host, dev, w) in enumerate(slot_bufs[1]):
                if direct and dev.shape[-1] == w:
                    dma.append(p)
                    continue
                hv = host.numpy()
                for i, (r, d) in enumerate(frames):
                    jobs.append((hv[0, i, :, :w], r[p] if nplanes == 3 else r))
                    jobs.append((hv[1, i, :, :w], d[p] if nplanes == 3 else d))
            if jobs:
                list(self._copier.map(_copy_into, jobs))
            with warnings.catch_warnings():  # read-only mappings: torch only reads them
                warnings.simplefilter("ignore", UserWarning)
                for p, (host, dev, w) in enumerate(slot_bufs[1]):
                    if p in dma:
                        for i, (r, d) in enumerate(frames):
                            dev[0, i].copy_(torch.from_numpy(r[p] if nplanes == 3 else r), non_blocking=True)
                            dev[1, i].copy_(torch.from_numpy(d[p] if nplanes == 3 else d), non_blocking=True)
                    else:
                        dev.copy_(host, non_blocking=True)
                    nbytes += dev.numel() * dev.element_size()
                    planes_ref.append(dev[0, :, :, :w])
                    planes_dist.append(dev[1, :, :, :w])
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        self._events[slot] = ev
        return planes_ref, planes_dist, ev, nbytes

    def _score_batch(self, planes_ref, planes_dist):
        cfg = self.config
        if self.color_weights is not None:
            return B.color_batch(planes_ref, planes_dist, cfg, weights=self.color_weights), None
        from . import engine

        pair = engine.device_pair(planes_ref[0], planes_dist[0], cfg.bit_depth, cfg.window.shape == "gauss")
        rec = luma_records(pair, cfg, strict=False)
        return rec.score, rec

    def score(self, ref_frames: Iterable, dist_frames: Iterable, direct: bool = False) -> SequenceResult:
        """Score two frame streams.  ``direct`` declares the planes page-locked
        (``FrameSource.pin``), enabling copy-free DMA staging."""
        torch = nat.torch_mod()
        result = SequenceResult()
        pending = []
        batch: list = []
        slot = 0
        compute = torch.cuda.current_stream(self.device)

        def flush(frames):
            nonlocal slot
            pr, pd, ev, nbytes = self._stage(slot, frames, direct)
            result.h2d_bytes += nbytes
            compute.wait_event(ev)
            score, terms = self._score_batch(pr, pd)
            done = torch.cuda.Event()
            done.record(compute)
            self._done[slot] = done
            pending.append((len(frames), score, terms))
            slot ^= 1

        for r, d in zip(ref_frames, dist_frames):
            batch.append((r, d))
            if len(batch) == self.batch_frames:
                flush(batch)
                batch = []
        if batch:
            flush(batch)
        idx = 0
        for count, score, rec in pending:
            s = score.cpu().numpy()
            extra = [None if t is None else t.cpu().numpy() for t in
                     ((rec.am, rec.l_mean, rec.cs_mean) if rec is not None else (None, None, None))]
            for i in range(count):
                am, lm, cm = (None if e is None else float(e[i]) for e in extra)
                result.records.append(FrameRecord(idx, float(s[i]), am, lm, cm))
                idx += 1
        if self.config.spatial_pool.startswith("cov") and np.isnan(result.scores).any():
            from .errors import ZeroMeanCoV

            raise ZeroMeanCoV("coefficient of variation is undefined for a zero-mean quality map")
        if not result.records:
            raise EmptySeries("no frames to score")
        result.pooled = pool_temporal(ScoreSeries(result.scores), self.config.temporal_pool)
        return result


def score_sequence(ref_frames, dist_frames, config: SsimConfig = SsimConfig(), batch_frames: int = 16,
                   color_weights=None) -> SequenceResult:
    """Convenience wrapper around ``SequenceScorer``."""
    return SequenceScorer(config, batch_frames, color_weights).score(ref_frames, dist_frames)
