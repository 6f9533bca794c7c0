"""Device-side orchestration: marshal planes to HBM and call the C ABI.

Every public scoring function of the package funnels into the handful of
calls below, which launch the hand-written sm_100a kernels in libssimk.so on
the current torch CUDA stream.  Host arrays are uploaded once (pinned staging,
16-byte aligned pitches); device tensors are used in place when their layout
already satisfies the kernels' alignment contract.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as nat
from .errors import ValidationError


@dataclass
class DevicePair:
    """A batch [n, h, w] of ref/dist frames resident in HBM, kernel-ready."""

    ref: "object"
    dist: "object"
    code: int
    bit_depth: int
    scale_log2: int = 0

    @property
    def shape(self):
        return tuple(self.ref.shape)

    def planes(self) -> nat.Planes:
        return nat.make_planes(self.ref, self.dist, self.code, self.bit_depth, self.scale_log2)


# ---------------------------------------------------------------------------
# host -> device
# ---------------------------------------------------------------------------

def _classify(a: np.ndarray, want_gauss: bool) -> tuple[np.dtype, int]:
    """Storage dtype + C-ABI code for a host sample array."""
    if a.dtype == np.uint8:
        return np.dtype(np.uint8), nat.U8
    if a.dtype == np.uint16:  # fits u16 by type: no range scan
        return np.dtype(np.uint16), nat.U16
    if a.dtype.kind in "ui":
        lo, hi = int(a.min()), int(a.max())
        if lo >= 0 and hi <= 255 and a.dtype.itemsize == 1:
            return np.dtype(np.uint8), nat.U8
        if lo >= 0 and hi <= 0xFFFF:
            return np.dtype(np.uint16), nat.U16
        return (np.dtype(np.float32), nat.F32) if want_gauss else (np.dtype(np.float64), nat.F64)
    if a.dtype.kind == "b":
        return np.dtype(np.uint8), nat.U8
    if want_gauss:
        return np.dtype(np.float32), nat.F32
    return np.dtype(np.float64), nat.F64


def _effective_depth(arrs, code: int, bit_depth: int) -> int:
    """Bit depth that bounds the stored integer samples (selects u32/u64 sums)."""
    if code in (nat.U8, nat.U16):
        hi = max(int(a.max()) for a in arrs)
        return min(16, max(bit_depth, 8, hi.bit_length()))
    return bit_depth


def upload_pair(ref: np.ndarray, dist: np.ndarray, bit_depth: int, gauss: bool,
                device=None, stream=None, validated: bool = False) -> DevicePair:
    """Copy one or a batch of host frame pairs into aligned device buffers (on ``stream``, or
    the current stream).  ``validated``: the samples already passed the container range
    check (``LumaPlane``: integers in [0, 2^bit_depth - 1]), so ``bit_depth`` bounds them and
    no host scan is repeated here."""
    torch = nat.torch_mod()
    device = device or nat.require_device()
    a = np.asarray(ref)
    b = np.asarray(dist)
    if a.ndim == 2:
        a, b = a[None], b[None]
    dt_a, code_a = _classify(a, gauss)
    dt_b, code_b = _classify(b, gauss)
    # both frames of a pair share one storage type (the kernels take one dtype)
    order = [nat.U8, nat.U16, nat.F32, nat.F64]
    code = max(code_a, code_b, key=order.index)
    np_dt = {nat.U8: np.uint8, nat.U16: np.uint16, nat.F32: np.float32, nat.F64: np.float64}[code]
    n, h, w = a.shape
    pitch = nat.aligned_pitch(w, code)
    t_dt = {nat.U8: torch.uint8, nat.U16: torch.uint16, nat.F32: torch.float32, nat.F64: torch.float64}[code]
    host = torch.empty((2, n, h, pitch), dtype=t_dt, pin_memory=True)
    hv = host.numpy()
    hv[0, :, :, :w] = a
    hv[1, :, :, :w] = b
    if pitch > w:
        hv[:, :, :, w:] = 0
    if stream is not None:
        with torch.cuda.stream(stream):
            dev = host.to(device, non_blocking=True)
    else:
        dev = host.to(device, non_blocking=True)
    depth = (max(8, min(16, bit_depth)) if validated and code in (nat.U8, nat.U16)
             else _effective_depth((a, b), code, bit_depth))
    return DevicePair(dev[0, :, :, :w], dev[1, :, :, :w], code, depth)


def device_pair(ref, dist, bit_depth: int, gauss: bool, scale_log2: int = 0) -> DevicePair:
    """Wrap [n,h,w] (or [h,w]) CUDA tensors, re-laying them out only if misaligned."""
    torch = nat.torch_mod()
    if ref.shape != dist.shape:
        from .errors import DimensionMismatch

        raise DimensionMismatch(f"reference is {tuple(ref.shape)}, distorted is {tuple(dist.shape)}")
    if ref.dim() == 2:
        ref, dist = ref.unsqueeze(0), dist.unsqueeze(0)
    if ref.dim() != 3:
        raise ValidationError("device batches must be [n, h, w] tensors")
    if not ref.is_cuda or not dist.is_cuda:
        raise ValidationError("device batches must be CUDA tensors")
    if ref.dtype != dist.dtype:
        raise ValidationError(f"ref/dist dtypes differ: {ref.dtype} vs {dist.dtype}")
    if ref.dtype == torch.float64 and gauss:
        ref, dist = ref.float(), dist.float()
    code = nat.dtype_code(ref)
    es = nat.esize(code)

    def ok(t) -> bool:
        return (t.stride(2) == 1 and (t.data_ptr() % 16) == 0 and (t.stride(1) * es) % 16 == 0
                and (t.stride(0) * es) % 16 == 0 and t.stride(0) >= t.stride(1) * t.shape[1])

    if not (ok(ref) and ok(dist) and ref.stride() == dist.stride()):
        n, h, w = ref.shape
        pitch = nat.aligned_pitch(w, code)
        buf = torch.zeros((2, n, h, pitch), dtype=ref.dtype, device=ref.device)
        buf[0, :, :, :w].copy_(ref)
        buf[1, :, :, :w].copy_(dist)
        ref, dist = buf[0, :, :, :w], buf[1, :, :, :w]
    return DevicePair(ref, dist, code, bit_depth, scale_log2)


# ---------------------------------------------------------------------------
# kernels
# ---------------------------------------------------------------------------

def _ptr(t, row: int = 0) -> Optional[int]:
    return None if t is None else t[row:].data_ptr()


def grid_shape(h: int, w: int, k: int, s: int) -> tuple[int, int]:
    return (h - k) // s + 1, (w - k) // s + 1


def ssim(pair: DevicePair, window, c1: float, c2: float, want: int, stream=None):
    """Fused SSIM over a device batch.

    Returns (sums [n,3] float64 device tensor (sum q, sum l, sum cs; a 4th column sum q^2
    with SSK_WANT_Q2), maps or None).
    Maps: SSK_MAP_TERMS -> [n,3,gh,gw] (l, cs, q); SSK_MAP_STATS -> [n,5,gh,gw];
    float32 for Gaussian windows (float64 with SSK_MAP_F64: the fp64 kernel), float64 for
    rect windows.
    """
    torch = nat.torch_mod()
    lib = nat.lib()
    n, h, w = pair.shape
    planes = pair.planes()
    win = nat.make_window(window, c1, c2)
    dev = pair.ref.device
    sums = torch.empty((n, 4 if want & nat.WANT_Q2 else 3), dtype=torch.float64, device=dev)
    maps = None
    if want & (nat.MAP_TERMS | nat.MAP_STATS):
        gh, gw = grid_shape(h, w, window.k, window.stride)
        nplanes = 5 if want & nat.MAP_STATS else 3
        mdt = torch.float32 if window.shape == "gauss" and not want & nat.MAP_F64 else torch.float64
        maps = torch.empty((n, nplanes, gh, gw), dtype=mdt, device=dev)
    ws_bytes = lib.ssk_ssim_workspace_bytes(ctypes.byref(planes), ctypes.byref(win))
    if ws_bytes == 0:
        # surface the precise validation error
        nat.raise_for(lib.ssk_ssim(ctypes.byref(planes), ctypes.byref(win), want, sums.data_ptr(),
                                   _ptr(maps), None, 0, nat.stream_handle(stream)), "ssim")
    ws = nat.WORKSPACE.get(ws_bytes, dev, stream)
    rc = lib.ssk_ssim(ctypes.byref(planes), ctypes.byref(win), want, sums.data_ptr(), _ptr(maps),
                      ws.data_ptr(), ws.numel(), nat.stream_handle(stream))
    nat.raise_for(rc, "ssim")
    return sums, maps


# Batches of at least this many frames run as two halves on two side streams, so the
# last (partial) wave of each kernel of one half is filled by CTAs of the other half
# (measured on 64 x 1080p: 1.007 -> 0.983 ms per MS-SSIM step).  Per-frame results
# do not depend on the split (segmentation depends on the frame geometry only).
SPLIT_MIN_FRAMES = 32
_DEFAULT_PARTS = int(os.environ.get("SSK_MSSSIM_PARTS", "2"))  # A/B switch: sub-batches of a large batch
_SIDE_STREAMS: dict = {}


def _side_streams(device, count: int):
    torch = nat.torch_mod()
    key = device.index
    have = _SIDE_STREAMS.get(key, [])
    prio = int(os.environ.get("SSK_SIDE_PRIORITY", "0"))
    while len(have) < count:
        # optionally the first half's stream at high priority: its coarse levels get CTA
        # slots ahead of the second half's level-0 tiles as SMs free up (helped the persistent
        # level-0 kernel, 0.897 -> 0.892 ms; with the classic two-CTAs-per-SM level-0 kernel
        # equal priorities measure 0.866 vs 0.911 ms per step, so it is off by default)
        have.append(torch.cuda.Stream(device=device, priority=-1 if (prio and not have) else 0))
    _SIDE_STREAMS[key] = have
    return have[:count]


def msssim_levels(pair: DevicePair, window, c1: float, c2: float, levels: int,
                  with_ssim: bool = False, spec=None, stream=None, split: Optional[int] = None):
    """Whole MS-SSIM pyramid in one library call (two, on side streams, for large batches).

    Returns (level means [n, levels] (cs below the coarsest, q at it), combined
    score [n] or None (when ``spec`` is given), level-0 SSIM means (q, l, cs)
    [n, 3] or None).
    """
    torch = nat.torch_mod()
    lib = nat.lib()
    n, h, w = pair.shape
    win = nat.make_window(window, c1, c2)
    dev = pair.ref.device
    means = torch.empty((n, levels), dtype=torch.float64, device=dev)
    ssim_sums = torch.empty((n, 3), dtype=torch.float64, device=dev) if with_ssim else None
    scores = None
    exps = None
    agg = 0
    if spec is not None:
        scores = torch.empty((n,), dtype=torch.float64, device=dev)
        e = spec.effective_exponents()
        exps = (ctypes.c_double * len(e))(*e)
        agg = 2 if spec.aggregation == "sum" else 1

    def run(part: DevicePair, lo: int, st) -> None:
        planes = part.planes()
        ws_bytes = lib.ssk_msssim_workspace_bytes(ctypes.byref(planes), ctypes.byref(win), levels)
        ws = nat.WORKSPACE.get(max(ws_bytes, 256), dev, st)
        rc = lib.ssk_msssim(ctypes.byref(planes), ctypes.byref(win), levels, exps, agg,
                            means[lo:].data_ptr(), _ptr(scores, lo), _ptr(ssim_sums, lo), ws.data_ptr(), ws.numel(),
                            nat.stream_handle(st))
        nat.raise_for(rc, "msssim")

    parts = split if split is not None else (_DEFAULT_PARTS if n >= SPLIT_MIN_FRAMES else 1)
    parts = max(1, min(int(parts), n))
    if parts == 1:
        run(pair, 0, stream)
        return means, scores, ssim_sums
    caller = stream if stream is not None else torch.cuda.current_stream(dev)
    ready = torch.cuda.Event()
    ready.record(caller)
    bounds = [round(i * n / parts) for i in range(parts + 1)]
    sides = _side_streams(dev, parts)
    for i, side in enumerate(sides):
        lo, hi = bounds[i], bounds[i + 1]
        side.wait_event(ready)  # inputs and outputs were produced / allocated on the caller's stream
        run(DevicePair(pair.ref[lo:hi], pair.dist[lo:hi], pair.code, pair.bit_depth, pair.scale_log2), lo, side)
    for side in sides:
        caller.wait_stream(side)
    return means, scores, ssim_sums


def window_sums(pair: DevicePair, k: int, stride: int, stream=None):
    """Exact int64 window sums [n, 5, gh, gw] of (x, y, x^2, y^2, xy)."""
    torch = nat.torch_mod()
    lib = nat.lib()
    n, h, w = pair.shape
    gh, gw = grid_shape(h, w, k, stride)
    out = torch.empty((n, 5, gh, gw), dtype=torch.int64, device=pair.ref.device)
    planes = pair.planes()
    win = nat.Window(shape=nat.RECT, k=k, stride=stride, _pad=0, c1=1.0, c2=1.0)
    ws_bytes = lib.ssk_ssim_workspace_bytes(ctypes.byref(planes), ctypes.byref(win))
    ws = nat.WORKSPACE.get(max(ws_bytes, 256), pair.ref.device, stream)
    rc = lib.ssk_box_window_sums(ctypes.byref(planes), k, stride, out.data_ptr(), ws.data_ptr(),
                                 ws.numel(), nat.stream_handle(stream))
    nat.raise_for(rc, "window sums")
    return out


def integral_tables(pair: DevicePair, stream=None):
    """Five summed-area tables [n, 5, h+1, w+1] (int64 for integer samples, else float64)."""
    torch = nat.torch_mod()
    n, h, w = pair.shape
    integer = pair.code in (nat.U8, nat.U16, nat.U32)
    out = torch.empty((n, 5, h + 1, w + 1), dtype=torch.int64 if integer else torch.float64,
                      device=pair.ref.device)
    rc = nat.lib().ssk_integral_tables(ctypes.byref(pair.planes()), out.data_ptr(), nat.stream_handle(stream))
    nat.raise_for(rc, "integral tables")
    return out


def downsample(pair: DevicePair, stream=None) -> DevicePair:
    """One 2x2 pyramid step of both frames (exact scaled integers or float)."""
    torch = nat.torch_mod()
    n, h, w = pair.shape
    h2, w2 = h // 2, w // 2
    if pair.code in (nat.F32, nat.F64):
        code, scale = pair.code, pair.scale_log2
    else:
        top = ((1 << pair.bit_depth) - 1) << (pair.scale_log2 + 2)
        code = nat.U16 if top <= 0xFFFF else nat.U32
        scale = pair.scale_log2 + 2
    t_dt = {nat.U16: torch.uint16, nat.U32: torch.uint32, nat.F32: torch.float32, nat.F64: torch.float64}[code]
    pitch = nat.aligned_pitch(max(w2, 1), code)
    buf = torch.empty((2, n, max(h2, 1), pitch), dtype=t_dt, device=pair.ref.device)
    rc = nat.lib().ssk_downsample(ctypes.byref(pair.planes()), buf[0].data_ptr(), buf[1].data_ptr(),
                                  code, pitch, max(h2, 1) * pitch, nat.stream_handle(stream))
    nat.raise_for(rc, "downsample")
    return DevicePair(buf[0, :, :h2, :w2], buf[1, :, :h2, :w2], code, pair.bit_depth, scale)


def to_float64(pair_tensor, code: int, scale_log2: int):
    """Device samples as float64 values (applies the 2^-scale of pyramid levels)."""
    torch = nat.torch_mod()
    t = pair_tensor
    if code in (nat.U16, nat.U32):
        t = t.to(torch.int64)
    v = t.to(torch.float64)
    return v * (2.0 ** -scale_log2) if scale_log2 else v


def frame_means(sums, count: int, stream=None):
    """sums / count with an IEEE division on the device (``ssk_divide``); every path derives
    means this way, so per-pair and batched scores are bit-identical."""
    torch = nat.torch_mod()
    src = sums.contiguous()
    out = torch.empty_like(src)
    nat.raise_for(nat.lib().ssk_divide(src.data_ptr(), src.numel(), float(count), out.data_ptr(),
                                       nat.stream_handle(stream)), "frame_means")
    return out


def launch_count() -> int:
    return int(nat.lib().ssk_launch_count())
