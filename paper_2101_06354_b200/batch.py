"""Batched device API: the throughput path (new API; the reference scores one pair per call).

All functions take [n, h, w] CUDA tensors (u8 / u16 / f32) already resident
in HBM, run one fused kernel launch per pyramid level over the whole batch and
return per-frame float64 results as device tensors; nothing but per-frame
scalars is produced.  The semantics per frame are exactly those of
``ssim_score`` / ``msssim`` / ``fixed_weight_cssim`` / ``channelwise_cssim``
(src/ssim.py:68-70, src/multiscale.py:77-90, src/color.py:119-141), and the
per-frame record matches the pipeline's ``FrameScore`` fields
(score, am, l_mean, cs_mean; src/pipeline.py:57-58, :230-236).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

from . import _native as nat
from . import engine
from .errors import TooManyLevels, ValidationError
from .moments import check_fit, resolve_engine
from .options import MultiscaleSpec, SsimConfig


@dataclass
class FrameTerms:
    """Per-frame mean q (== score / am), mean l and mean cs, each a [n] float64 device tensor."""

    score: "object"
    l_mean: "object"
    cs_mean: "object"


def _pair(ref, dist, config: SsimConfig) -> engine.DevicePair:
    pair = engine.device_pair(ref, dist, config.bit_depth, config.window.shape == "gauss")
    _, h, w = pair.shape
    check_fit(h, w, config.window.k)
    resolve_engine(config.window, config.engine)
    return pair


def ssim_terms_batch(ref, dist, config: SsimConfig = SsimConfig(), stream=None) -> FrameTerms:
    pair = _pair(ref, dist, config)
    _, h, w = pair.shape
    sums, _ = engine.ssim(pair, config.window, config.c1, config.c2,
                          nat.WANT_Q | nat.WANT_L | nat.WANT_CS, stream)
    gh, gw = engine.grid_shape(h, w, config.window.k, config.window.stride)
    means = engine.frame_means(sums, gh * gw, stream)
    return FrameTerms(means[:, 0], means[:, 1], means[:, 2])


def ssim_batch(ref, dist, config: SsimConfig = SsimConfig(), stream=None):
    """Mean SSIM per frame pair: [n] float64 on the device."""
    return ssim_terms_batch(ref, dist, config, stream).score


def msssim_batch(ref, dist, config: SsimConfig = SsimConfig(), spec: Optional[MultiscaleSpec] = None,
                 with_ssim: bool = False, stream=None):
    """MS-SSIM per frame pair ([n] float64 device tensor).

    With ``with_ssim`` the plain SSIM terms of scale 0 come from the same pass
    (returned as a second value, a ``FrameTerms``).
    """
    spec = MultiscaleSpec.product() if spec is None else spec
    if not spec.enabled:
        raise ValidationError("multiscale aggregation is off; use ssim_score instead")
    pair = _pair(ref, dist, config)
    _, h, w = pair.shape
    k = config.window.k
    if min(h, w) // (1 << (spec.levels - 1)) < k:
        raise TooManyLevels(f"a {k}x{k} window does not fit the coarsest of {spec.levels} scales of a {w}x{h} image")
    _, score, ssim_sums = engine.msssim_levels(pair, config.window, config.c1, config.c2, spec.levels,
                                               with_ssim=with_ssim, spec=spec, stream=stream)
    if not with_ssim:
        return score
    return score, FrameTerms(ssim_sums[:, 0], ssim_sums[:, 1], ssim_sums[:, 2])


def color_batch(planes_ref, planes_dist, config: SsimConfig = SsimConfig(), weights=None,
                alpha: Optional[float] = None, beta: Optional[float] = None, stream=None):
    """Channel-wise color SSIM per frame from three [n, h_c, w_c] device batches per side.

    ``weights`` -> fixed_weight_cssim; ``alpha``/``beta`` -> channelwise_cssim.
    Channels are scored at their own resolution (4:2:0 chroma stays 4:2:0).
    """
    if (weights is None) == (alpha is None):
        raise ValidationError("give either fixed weights or the cw alpha/beta pair")
    scores = [ssim_batch(a, b, config, stream) for a, b in zip(planes_ref, planes_dist)]
    if weights is not None:
        if abs(sum(weights) - 1.0) > 1e-9:
            raise ValidationError(f"channel weights must sum to 1, got {sum(weights)!r}")
        out = 0.0
        for wgt, s in zip(weights, scores):
            out = out + wgt * s
        return out
    denom = 1.0 + alpha + beta
    if abs(denom) < 1e-12:
        from .errors import DegenerateWeights

        raise DegenerateWeights("1 + alpha + beta must be nonzero")
    return (scores[0] + alpha * scores[1] + beta * scores[2]) / denom


class HostBatchScorer:
    """End-to-end scoring of frame batches held in (pinned) host memory.

    Each call uploads the batch in chunks on a copy stream, overlapping the
    H2D of chunk i+1 with the scoring of chunk i on the compute stream, and
    returns the per-frame scores on the host.  Device buffers are reused
    across calls (double-buffered chunks), so steady-state calls allocate
    nothing.  ``mode`` is "ssim", "msssim" or "both" (SSIM and MS-SSIM from
    one pyramid pass, scale 0 shared).
    """

    def __init__(self, config: SsimConfig = SsimConfig(), spec: Optional[MultiscaleSpec] = None,
                 mode: str = "both", chunk: int = 8, device=None):
        if mode not in ("ssim", "msssim", "both"):
            raise ValidationError(f"unknown mode {mode!r}")
        torch = nat.torch_mod()
        self.config, self.mode, self.chunk = config, mode, max(1, int(chunk))
        self.spec = MultiscaleSpec.product() if spec is None else spec
        self.device = device or nat.require_device()
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self._bufs = {}
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def _buffers(self, slot, like):
        torch = nat.torch_mod()
        key = (slot, tuple(like.shape[1:]), like.dtype)
        buf = self._bufs.get(key)
        if buf is None or buf[0].shape[0] < self.chunk:
            buf = (torch.empty((self.chunk, *like.shape[1:]), dtype=like.dtype, device=self.device),
                   torch.empty((self.chunk, *like.shape[1:]), dtype=like.dtype, device=self.device),
                   [None])
            self._bufs[key] = buf
        return buf

    def __call__(self, ref_host, dist_host):
        """ref_host/dist_host: [n, h, w] CPU tensors (pinned for async copies).

        Returns float64 numpy arrays: ``msssim`` -> [n]; ``ssim`` -> [n, 3]
        (score, l_mean, cs_mean); ``both`` -> ([n], [n, 3]).
        """
        return self.submit(ref_host, dist_host).result()

    def submit(self, ref_host, dist_host) -> "PendingScores":
        """Queue one batch without waiting for it: uploads, kernels and the score read-back
        are enqueued and a handle is returned whose ``result()`` waits for this batch only.
        A stream of batches submitted one ahead keeps the copy engine busy across batches
        (the next batch's uploads overlap this batch's last chunk and read-back)."""
        torch = nat.torch_mod()
        n = ref_host.shape[0]
        compute = torch.cuda.current_stream(self.device)
        outs_ms, outs_ss = [], []
        self.h2d_bytes = self.d2h_bytes = 0
        for ci, start in enumerate(range(0, n, self.chunk)):
            stop = min(n, start + self.chunk)
            r_dev, d_dev, done = self._buffers(ci & 1, ref_host)
            with torch.cuda.stream(self.copy_stream):
                if done[0] is not None:
                    self.copy_stream.wait_event(done[0])
                r_dev[: stop - start].copy_(ref_host[start:stop], non_blocking=True)
                d_dev[: stop - start].copy_(dist_host[start:stop], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
            self.h2d_bytes += 2 * ref_host[start:stop].numel() * ref_host.element_size()
            compute.wait_event(ev)
            r, d = r_dev[: stop - start], d_dev[: stop - start]
            if self.mode == "ssim":
                t = ssim_terms_batch(r, d, self.config)
                outs_ss.append(torch.stack([t.score, t.l_mean, t.cs_mean], dim=1))
            else:
                res = msssim_batch(r, d, self.config, self.spec, with_ssim=self.mode == "both")
                if self.mode == "both":
                    ms, t = res
                    outs_ss.append(torch.stack([t.score, t.l_mean, t.cs_mean], dim=1))
                else:
                    ms = res
                outs_ms.append(ms)
            fin = torch.cuda.Event()
            fin.record(compute)
            done[0] = fin

        def to_host(outs):
            if not outs:
                return None
            dev = torch.cat(outs)
            host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
            host.copy_(dev, non_blocking=True)
            return host

        ms_host, ss_host = to_host(outs_ms), to_host(outs_ss)
        ready = torch.cuda.Event()
        ready.record(compute)
        self.d2h_bytes = sum(0 if t is None else t.numel() * t.element_size() for t in (ms_host, ss_host))
        return PendingScores(self.mode, ms_host, ss_host, ready)


class PendingScores:
    """Scores of a submitted batch (``HostBatchScorer.submit``); ``result()`` waits for them."""

    def __init__(self, mode: str, ms_host, ss_host, ready):
        self.mode, self._ms, self._ss, self._ready = mode, ms_host, ss_host, ready

    def done(self) -> bool:
        return self._ready.query()

    def result(self):
        self._ready.synchronize()
        ms = None if self._ms is None else self._ms.numpy()
        ss = None if self._ss is None else self._ss.numpy()
        if self.mode == "msssim":
            return ms
        if self.mode == "ssim":
            return ss
        return ms, ss
