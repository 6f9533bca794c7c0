"""Seeded synthetic frame pairs for the five BASELINE.json configurations.

The reference measures on no public dataset for this path (BASELINE.json
"published": {}; the paper's subjective databases are not needed for
throughput), so seeded synthetic inputs with the configurations' shapes,
bit depths and distortion types stand in.  Every frame i of
config c is generated from ``SeedSequence(BASE[c]).spawn`` child i, so any
shard (GPU rank, CPU worker) can regenerate exactly its own frames.
"""

from __future__ import annotations

import numpy as np

BASE = {1: 101, 2: 202, 3: 303, 4: 404, 5: 505}


def _child(config: int, index: int) -> np.random.Generator:
    ss = np.random.SeedSequence(BASE[config])
    return np.random.default_rng(ss.spawn(index + 1)[index])


def inv_f_noise(rng: np.random.Generator, h: int, w: int, peak: float) -> np.ndarray:
    """1/f-spectrum noise: complex N(0,1) spectrum / |f| (DC weight 1), real(ifft2), min-max to [0, peak]."""
    spec = rng.standard_normal((h, w)) + 1j * rng.standard_normal((h, w))
    fy = np.fft.fftfreq(h)[:, None]
    fx = np.fft.fftfreq(w)[None, :]
    mag = np.sqrt(fx * fx + fy * fy)
    mag[0, 0] = 1.0
    field = np.real(np.fft.ifft2(spec / mag))
    lo, hi = field.min(), field.max()
    return np.round((field - lo) / (hi - lo) * peak)


def blur_reflect(img: np.ndarray, sigma: float) -> np.ndarray:
    """Separable Gaussian blur, reflect padding, radius ceil(3 sigma)."""
    r = int(np.ceil(3 * sigma))
    x = np.arange(-r, r + 1, dtype=np.float64)
    g = np.exp(-(x * x) / (2 * sigma * sigma))
    g /= g.sum()
    p = np.pad(img, r, mode="reflect")
    h, w = img.shape
    rows = sum(g[i] * p[i:i + h, :] for i in range(g.size))
    return sum(g[j] * rows[:, j:j + w] for j in range(g.size))


def dct_quantise(ref: np.ndarray, step: float) -> np.ndarray:
    """8x8-block orthonormal DCT-II quantisation of (ref - 128), uniform step."""
    from scipy.fft import dctn, idctn

    h, w = ref.shape
    blocks = (ref.astype(np.float64) - 128.0).reshape(h // 8, 8, w // 8, 8)
    coef = dctn(blocks, axes=(1, 3), norm="ortho")
    coef = np.round(coef / step) * step
    out = idctn(coef, axes=(1, 3), norm="ortho").reshape(h, w) + 128.0
    return np.clip(np.round(out), 0, 255).astype(np.uint8)


def config1_pair() -> tuple[np.ndarray, np.ndarray]:
    """512x512 u8: blurred white noise (sigma 2) vs + N(0, 10)."""
    rng = _child(1, 0)
    ref = blur_reflect(rng.standard_normal((512, 512)), 2.0)
    lo, hi = ref.min(), ref.max()
    ref = np.round((ref - lo) / (hi - lo) * 255.0).astype(np.uint8)
    dist = np.clip(np.round(ref + rng.normal(0.0, 10.0, ref.shape)), 0, 255).astype(np.uint8)
    return ref, dist


def dct_pair(config: int, index: int, h: int = 1080, w: int = 1920) -> tuple[np.ndarray, np.ndarray]:
    """Configs 2 / 5: u8 1/f noise vs its DCT quantisation with step ~ U[4, 40]."""
    rng = _child(config, index)
    ref = inv_f_noise(rng, h, w, 255.0).astype(np.uint8)
    step = rng.uniform(4.0, 40.0)
    return ref, dct_quantise(ref, step)


def config4_pair(index: int, h: int = 2160, w: int = 3840) -> tuple[np.ndarray, np.ndarray]:
    """10-bit in u16: 1/f noise vs bicubic x1/2 -> x2 + N(0, 8), clipped to [0, 1023]."""
    import torch

    rng = _child(4, index)
    ref = inv_f_noise(rng, h, w, 1023.0)
    t = torch.from_numpy(ref)[None, None]
    small = torch.nn.functional.interpolate(t, scale_factor=0.5, mode="bicubic", align_corners=False)
    up = torch.nn.functional.interpolate(small, size=(h, w), mode="bicubic", align_corners=False)[0, 0].numpy()
    dist = np.clip(np.round(up + rng.normal(0.0, 8.0, up.shape)), 0, 1023)
    return ref.astype(np.uint16), dist.astype(np.uint16)


class VideoConfig3:
    """300 frames of 1080p YUV420 8-bit: translating 1/f content vs blur + noise."""

    def __init__(self, frames: int = 300, h: int = 1080, w: int = 1920):
        self.frames, self.h, self.w = frames, h, w
        rng = _child(3, 0)
        self.y_base = inv_f_noise(rng, h, w + 2 * (frames - 1), 255.0)
        self.cb_base = inv_f_noise(rng, h // 2, w // 2 + frames - 1, 255.0)
        self.cr_base = inv_f_noise(rng, h // 2, w // 2 + frames - 1, 255.0)

    def pair(self, t: int):
        from scipy.ndimage import gaussian_filter

        rng = _child(3, t + 1)
        sigma = rng.uniform(0.5, 2.0)
        ref = (self.y_base[:, 2 * t:2 * t + self.w], self.cb_base[:, t:t + self.w // 2],
               self.cr_base[:, t:t + self.w // 2])
        out_r, out_d = [], []
        for plane in ref:
            d = gaussian_filter(plane, sigma) + rng.normal(0.0, 5.0, plane.shape)
            out_r.append(np.ascontiguousarray(plane).astype(np.uint8))
            out_d.append(np.clip(np.round(d), 0, 255).astype(np.uint8))
        return tuple(out_r), tuple(out_d)
