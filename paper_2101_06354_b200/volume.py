"""SSIM-3D over k x k x Kt neighbourhoods with rolling temporal sums (ssimkit src/spatiotemporal.py).

Device-resident ``RollingVolume``: the last Kt frame pairs stay in HBM, the
five temporal-sum planes (x, y, x^2, y^2, xy) are updated per pushed frame by
one kernel (T += I(new) - I(old), src/spatiotemporal.py:84-90), and the spatial
k x k window runs on the exact running-sum box kernel with area = k^2 * depth
(:116-138).  Integer frames use int64 planes: the recursion is exact, so the
reference's periodic refresh (REFRESH_INTERVAL) changes nothing and results
equal the reference's float64 sums (also exact integers) bit for bit.  Float
frames use float64 planes updated in the reference's order and refreshed from
the buffer every ``refresh_interval`` pushes, like the reference.  Per-frame
cost is independent of Kt (the reference's acceptance criterion C4).
"""

from __future__ import annotations

import ctypes
from collections import deque
from typing import Iterable, Optional

import numpy as np

from . import _native as nat
from . import engine
from .errors import DimensionMismatch, GaussianNotSupported3D, ValidationError
from .moments import LocalStatsMaps
from .options import MultiscaleSpec, SsimConfig, WindowSpec
from .planes import PlaneLike, QualityMap, ScoreSeries, plane_data, validate_frame_pair
from .pyramid import combine_scale_scores, dyadic_downsample, msssim
from .scoring import SsimTermMaps

REFRESH_INTERVAL = 300


class RollingVolume:
    """Ring of the last Kt frame pairs (device) plus their five running sums (device)."""

    def __init__(self, kt: int, refresh_interval: int = REFRESH_INTERVAL):
        if not isinstance(kt, int) or isinstance(kt, bool) or kt < 1:
            raise ValidationError(f"temporal window must be an integer >= 1, got {kt!r}")
        self.kt = kt
        self.refresh_interval = refresh_interval
        self._buffer: deque = deque()
        self._planes = None
        self._is_float: Optional[bool] = None
        self._code: Optional[int] = None
        self._dims: Optional[tuple[int, int]] = None
        self._pushes = 0
        self._copy_stream = None

    @property
    def depth(self) -> int:
        return len(self._buffer)

    @property
    def buffer_planes(self) -> tuple[int, int]:
        return len(self._buffer), 0 if self._planes is None else 5

    # -- state -------------------------------------------------------------
    def _volume(self) -> nat.Volume:
        h, w = self._dims
        return nat.Volume(planes=self._planes.data_ptr(), is_float=int(self._is_float), h=h, w=w,
                          depth=max(1, self.depth), pitch=self._planes.stride(1))

    def _upload(self, a: np.ndarray):
        torch = nat.torch_mod()
        dev = nat.require_device()
        dt = np.float64 if self._is_float else (np.uint8 if self._code == nat.U8 else np.uint16)
        src = a if (a.dtype == dt and a.flags.c_contiguous) else np.ascontiguousarray(a, dtype=dt)
        # staged through a pinned buffer and copied asynchronously on the current stream
        tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.uint8): torch.uint8,
               np.dtype(np.uint16): torch.uint16}[src.dtype]
        host = torch.empty(src.shape, dtype=tdt, pin_memory=True)
        host.numpy()[...] = src
        return host.to(dev, non_blocking=True)

    def push(self, ref: PlaneLike, dist: PlaneLike, staged=None) -> "RollingVolume":
        """Advance the temporal window by one frame pair (src/spatiotemporal.py:60-97)."""
        torch = nat.torch_mod()
        ref, dist = validate_frame_pair(ref, dist)
        a, b = plane_data(ref), plane_data(dist)
        u8 = a.dtype == np.uint8 and b.dtype == np.uint8  # in range by type: no sample scans
        if self._dims is None:
            self._dims = a.shape
            ints = u8 or (a.dtype.kind in "ui" and b.dtype.kind in "ui" and min(a.min(), b.min()) >= 0)
            hi = 255 if u8 else (max(int(a.max()), int(b.max())) if ints else 0)
            self._is_float = not (ints and hi <= 0xFFFF)
            small = a.dtype == np.uint8 and b.dtype == np.uint8
            self._code = nat.F64 if self._is_float else (nat.U8 if small else nat.U16)
            h, w = self._dims
            dt = torch.float64 if self._is_float else torch.int64
            self._planes = torch.zeros((5, h, w), dtype=dt, device=nat.require_device())
        elif a.shape != self._dims:
            raise DimensionMismatch(f"frame {a.shape[::-1]} pushed into a {self._dims[::-1]} volume")
        elif not (u8 and not self._is_float):
            if not self._is_float:
                ints = a.dtype.kind in "ui" and b.dtype.kind in "ui"
                hi = max(int(a.max()), int(b.max())) if ints else 1 << 20
                if not ints or min(a.min(), b.min()) < 0 or hi > (255 if self._code == nat.U8 else 0xFFFF):
                    raise ValidationError("frames of one volume must keep the sample type of the first frame")
        if staged is not None and not self._is_float and staged[0].dtype == (
                torch.uint8 if self._code == nat.U8 else torch.uint16):
            # pre-staged pinned copies (ssim3d_series' prefetch pool): DMA on a side copy
            # stream so the upload of this frame overlaps the previous frame's kernels
            dev = nat.require_device()
            if self._copy_stream is None:
                self._copy_stream = torch.cuda.Stream(device=dev)
            cur = torch.cuda.current_stream(dev)
            with torch.cuda.stream(self._copy_stream):  # destination allocated on the copy stream
                ra, rb = staged[0].to(dev, non_blocking=True), staged[1].to(dev, non_blocking=True)
            cur.wait_stream(self._copy_stream)  # the kernels on `cur` see the frame
            ra.record_stream(cur)  # freed blocks are reused only after `cur` is done with them
            rb.record_stream(cur)
        else:
            ra, rb = self._upload(a), self._upload(b)
        lib = nat.lib()
        vol = self._volume()
        if self.depth == 0 or self.kt == 1:
            mode, old = 0, (None, None)
        elif self.depth == self.kt:
            mode, old = 2, self._buffer[0]
        else:
            mode, old = 1, (None, None)
        rc = lib.ssk_volume_update(ctypes.byref(vol), ra.data_ptr(), rb.data_ptr(),
                                   None if old[0] is None else old[0].data_ptr(),
                                   None if old[1] is None else old[1].data_ptr(),
                                   self._code, ra.stride(0), mode, nat.stream_handle())
        nat.raise_for(rc, "volume update")
        if self.depth == self.kt:
            self._buffer.popleft()
        self._buffer.append((ra, rb))
        self._pushes += 1
        if self.refresh_interval and self._pushes % self.refresh_interval == 0:
            self._refresh()
        return self

    def _refresh(self) -> None:
        """Rebuild the sums from the buffer (float volumes; integer sums are exact anyway)."""
        if not self._is_float:
            return
        n = self.depth
        refs = (ctypes.c_void_p * n)(*[r.data_ptr() for r, _ in self._buffer])
        dists = (ctypes.c_void_p * n)(*[d.data_ptr() for _, d in self._buffer])
        rc = nat.lib().ssk_volume_refresh(ctypes.byref(self._volume()), refs, dists, n, nat.F64,
                                          self._buffer[0][0].stride(0), nat.stream_handle())
        nat.raise_for(rc, "volume refresh")

    def direct_sums(self) -> list:
        """Sums recomputed from scratch over the buffered frames (src/spatiotemporal.py:103-115),
        on the device into fresh planes: the drift check against ``temporal_sums``."""
        if not self._buffer:
            raise ValidationError("no frames buffered")
        torch = nat.torch_mod()
        fresh = torch.zeros_like(self._planes)
        h, w = self._dims
        vol = nat.Volume(planes=fresh.data_ptr(), is_float=int(self._is_float), h=h, w=w,
                         depth=max(1, self.depth), pitch=fresh.stride(1))
        lib = nat.lib()
        for i, (ra, rb) in enumerate(self._buffer):
            rc = lib.ssk_volume_update(ctypes.byref(vol), ra.data_ptr(), rb.data_ptr(), None, None, self._code,
                                       ra.stride(0), 0 if i == 0 else 1, nat.stream_handle())
            nat.raise_for(rc, "volume direct sums")
        return [p.double().cpu().numpy() for p in fresh]

    def temporal_sums(self) -> list:
        if self._planes is None:
            raise ValidationError("no frames buffered")
        return [p.double().cpu().numpy() for p in self._planes]

    # -- statistics --------------------------------------------------------
    def _run(self, window: WindowSpec, c1: float, c2: float, want: int):
        torch = nat.torch_mod()
        if window.shape != "rect":
            raise GaussianNotSupported3D("3-D statistics support rectangular windows only")
        if self._planes is None:
            raise ValidationError("no frames buffered")
        h, w = self._dims
        if window.k > h or window.k > w:
            raise ValidationError(f"{window.k}x{window.k} window does not fit a {w}x{h} frame")
        lib = nat.lib()
        vol = self._volume()
        win = nat.make_window(window, c1, c2)
        dev = self._planes.device
        sums = torch.empty((1, 3), dtype=torch.float64, device=dev)
        gh, gw = engine.grid_shape(h, w, window.k, window.stride)
        maps = None
        if want & (nat.MAP_TERMS | nat.MAP_STATS):
            maps = torch.empty((1, 5 if want & nat.MAP_STATS else 3, gh, gw), dtype=torch.float64, device=dev)
        ws_bytes = lib.ssk_volume_workspace_bytes(ctypes.byref(vol), ctypes.byref(win))
        ws = nat.WORKSPACE.get(max(ws_bytes, 256), dev)
        rc = lib.ssk_volume_ssim(ctypes.byref(vol), ctypes.byref(win), want, sums.data_ptr(),
                                 None if maps is None else maps.data_ptr(), ws.data_ptr(), ws.numel(),
                                 nat.stream_handle())
        nat.raise_for(rc, "volume ssim")
        return sums, maps, (gh, gw)

    def local_statistics(self, window: WindowSpec) -> LocalStatsMaps:
        """k x k x depth local statistics (src/spatiotemporal.py:116-138)."""
        _, maps, _ = self._run(window, 1.0, 1.0, nat.MAP_STATS)
        m = maps[0].cpu().numpy()
        return LocalStatsMaps(mu1=m[0], mu2=m[1], var1=m[2], var2=m[3], cov=m[4], window_size=window.k,
                              stride=window.stride, source_dims=self._dims)

    def terms_device(self, window: WindowSpec, config: SsimConfig):
        """(mean q, mean l, mean cs) of the current 3-D SSIM map as a [3] float64 device tensor
        (no synchronisation: a series reads all frames' terms back at once)."""
        sums, _, (gh, gw) = self._run(window, config.c1, config.c2, nat.WANT_Q | nat.WANT_L | nat.WANT_CS)
        return engine.frame_means(sums, gh * gw)[0]

    def terms(self, window: WindowSpec, config: SsimConfig) -> tuple[float, float, float]:
        """(mean q, mean l, mean cs) of the current 3-D SSIM map, fused (no map leaves the GPU)."""
        s = self.terms_device(window, config).cpu().numpy()
        return float(s[0]), float(s[1]), float(s[2])


def push_frame(vol: RollingVolume, ref: PlaneLike, dist: PlaneLike) -> RollingVolume:
    return vol.push(ref, dist)


def ssim3d_map(vol: RollingVolume, window: WindowSpec, config: SsimConfig = SsimConfig()) -> SsimTermMaps:
    """SSIM term maps over the volume's current temporal window (src/spatiotemporal.py:146-149)."""
    _, maps, _ = vol._run(window, config.c1, config.c2, nat.WANT_Q | nat.WANT_L | nat.WANT_CS | nat.MAP_TERMS)
    m = maps[0].cpu().numpy()
    geom = dict(stride=window.stride, source_dims=vol._dims)
    return SsimTermMaps(QualityMap(m[0], **geom), QualityMap(m[1], **geom), QualityMap(m[2], **geom))


def ssim3d_series(ref_frames: Iterable[PlaneLike], dist_frames: Iterable[PlaneLike], kt: int,
                  config: SsimConfig = SsimConfig()) -> ScoreSeries:
    """Per-frame mean 3-D SSIM of two aligned streams (src/spatiotemporal.py:159-171)."""
    torch = nat.torch_mod()
    vol = RollingVolume(kt)
    terms = []

    def stage(pair):  # worker thread: copy a u8 / u16 frame pair into pinned host memory
        out = []
        for p in pair:
            a = plane_data(p)
            if a.dtype not in (np.uint8, np.uint16):
                return None
            t = torch.empty(a.shape, dtype=torch.uint8 if a.dtype == np.uint8 else torch.uint16, pin_memory=True)
            t.numpy()[...] = a
            out.append(t)
        return tuple(out)

    # integer frames are staged into pinned memory a few frames ahead on a small thread pool
    # (numpy copies release the GIL), so uploads are asynchronous DMA and the host loop only
    # issues launches; scores are read back once, after the last frame
    from concurrent.futures import ThreadPoolExecutor

    pairs = iter(zip(ref_frames, dist_frames))
    ahead = deque()
    with ThreadPoolExecutor(4) as ex:
        def fill():
            while len(ahead) < 8:
                nxt = next(pairs, None)
                if nxt is None:
                    return
                ahead.append((nxt, ex.submit(stage, nxt)))

        fill()
        while ahead:
            (ref, dist), fut = ahead.popleft()
            fill()
            validate_frame_pair(ref, dist)
            vol.push(ref, dist, staged=fut.result())
            terms.append(vol.terms_device(config.window, config))
    if not terms:
        return ScoreSeries(np.asarray([], dtype=np.float64))
    return ScoreSeries(torch.stack(terms)[:, 0].cpu().numpy())


def shard_with_halo(n_frames: int, rank: int, world: int, kt: int) -> tuple[int, int, int]:
    """(first frame to push, first frame to score, stop) of ``rank``'s contiguous block:
    SSIM-3D shards need the Kt-1 frames before their block as a halo."""
    from .video import shard_bounds

    if not isinstance(kt, int) or kt < 1:
        raise ValidationError(f"temporal window must be an integer >= 1, got {kt!r}")
    start, stop = shard_bounds(n_frames, rank, world)
    return max(0, start - (kt - 1)), start, stop


def ssim3d_series_shard(ref_frames, dist_frames, kt: int, rank: int, world: int,
                        config: SsimConfig = SsimConfig()) -> ScoreSeries:
    """This rank's slice of ``ssim3d_series``: the halo frames are pushed unscored, then
    the rank's own frames are scored.  Concatenating every rank's slice in rank order
    gives the unsharded series (bit-exactly for integer frames, whose rolling sums are
    exact; float volumes refresh on their own push count)."""
    if len(ref_frames) != len(dist_frames):
        raise DimensionMismatch("reference and distorted streams differ in length")
    lo, start, stop = shard_with_halo(len(ref_frames), rank, world, kt)
    vol = RollingVolume(kt)
    scores = []
    for i in range(lo, stop):
        vol.push(ref_frames[i], dist_frames[i])
        if i >= start:
            scores.append(vol.terms(config.window, config)[0])
    return ScoreSeries(np.asarray(scores))


def msssim3d(ref_frames: Iterable[PlaneLike], dist_frames: Iterable[PlaneLike], kt: int,
             spec: Optional[MultiscaleSpec] = None, config: SsimConfig = SsimConfig()) -> ScoreSeries:
    """Multiscale 3-D SSIM, one rolling volume per scale (src/spatiotemporal.py:174-207)."""
    spec = MultiscaleSpec.product() if spec is None else spec
    if not spec.enabled:
        raise ValidationError("multiscale aggregation is off; use ssim3d_series instead")
    if kt == 1 and config.window.shape == "rect":  # one-frame volume = the 2-D window: framewise MS-SSIM
        return ScoreSeries(np.asarray([msssim(r, d, config, spec) for r, d in zip(ref_frames, dist_frames)]))
    volumes = [RollingVolume(kt) for _ in range(spec.levels)]
    scores = []
    for ref, dist in zip(ref_frames, dist_frames):
        validate_frame_pair(ref, dist)
        cur_ref, cur_dist = ref, dist
        per_scale = []
        for level in range(spec.levels):
            if level > 0:
                cur_ref, cur_dist = dyadic_downsample(cur_ref), dyadic_downsample(cur_dist)
            volumes[level].push(cur_ref, cur_dist)
            q, _, cs = volumes[level].terms(config.window, config)
            per_scale.append(q if level == spec.levels - 1 else cs)
        scores.append(combine_scale_scores(per_scale, spec))
    return ScoreSeries(np.asarray(scores))
