"""CPU ORACLE — test infrastructure only, never part of the product path.

A float64/int64 numpy restatement of the reference's SSIM hot path
(ssimkit, /root/reference/pkg/src/ssimkit), written independently of the
reference sources but replaying the same algorithms and the same arithmetic
order, so that its outputs are bit-identical to the reference's:

  gaussian_kernel ........ src/stats.py:30-44
  sat / integral_set ..... src/stats.py:66-71, :96-116   (int64 for integer samples)
  grid_window_sums ....... src/stats.py:130-141         (four-corner rule)
  sliding_sums ........... src/stats.py:144-164         (direct k^2 loops)
  moments_from_sums ...... src/stats.py:185-202
  local_statistics ....... src/stats.py:205-261         (engine resolution :223-228)
  term_maps .............. src/ssim.py:31-46
  dyadic_downsample ...... src/multiscale.py:19-33
  scale_scores / combine . src/multiscale.py:36-74
  channel_scores ......... src/color.py:111-153         (cw / fixed models)
  pool_temporal_am ....... src/pooling.py:254-255
  scale factors .......... src/adaptation.py:23-90      (256-line rule, dh, sast)
  box_downsample ......... src/adaptation.py:93-110     (block means, ragged edges)
  pool_spatial ........... src/pooling.py:157-243       (am cov md fns dw mink lw pp)
  luma_frame_record ...... src/pipeline.py:197-236      (scale -> stats -> pool record)
  color conversions ...... src/color.py:64-108          (BT.709 YCbCr, luma, 4:2:0 upsample)
  qssim .................. src/color.py:159-256         (quaternion windowed similarity)
  delta_e / cmssim ....... src/color.py:263-334         (opponent smoothing, CIELAB weights)
  hue / hssim ............ src/color.py:341-371

Parity pinning: tests/test_oracle_golden.py checks this module against
golden vectors produced by the reference itself (tests/golden/make_golden.py,
run in the build container where /root/reference is importable) and against
the reference tests' known-answer values.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this module.
"""

from __future__ import annotations

import math

import numpy as np

STANDARD_EXPONENTS = (0.0448, 0.2856, 0.3001, 0.2363, 0.1333)


def constants(bit_depth: int = 8, k1: float = 0.01, k2: float = 0.03) -> tuple[float, float]:
    """C1 = (k1 L)^2, C2 = (k2 L)^2 with L = 2^bd - 1 (src/config.py:267-285)."""
    peak = float((1 << bit_depth) - 1)
    return (k1 * peak) ** 2, (k2 * peak) ** 2


def default_gaussian_size(sigma: float) -> int:
    return 2 * math.ceil(3.0 * sigma) + 1


def gaussian_kernel(sigma: float, k: int | None = None) -> np.ndarray:
    if k is None:
        k = default_gaussian_size(sigma)
    c = np.arange(k, dtype=np.float64) - (k - 1) / 2.0
    g = np.exp(-(c * c) / (2.0 * sigma * sigma))
    outer = np.outer(g, g)
    return outer / outer.sum()


# ---------------------------------------------------------------------------
# window sums
# ---------------------------------------------------------------------------

def sat(values: np.ndarray) -> np.ndarray:
    """(h+1) x (w+1) summed-area table with a zero first row and column."""
    h, w = values.shape
    table = np.zeros((h + 1, w + 1), dtype=values.dtype)
    table[1:, 1:] = values.cumsum(axis=0).cumsum(axis=1)
    return table


def promote_pair(a: np.ndarray, b: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """int64 when both inputs are integer, else float64 (src/stats.py:101-106)."""
    if a.dtype.kind in "ui" and b.dtype.kind in "ui":
        return a.astype(np.int64), b.astype(np.int64)
    return a.astype(np.float64), b.astype(np.float64)


def integral_set(a: np.ndarray, b: np.ndarray) -> dict:
    x, y = promote_pair(np.asarray(a), np.asarray(b))
    return {"sum1": sat(x), "sum2": sat(y), "sq1": sat(x * x), "sq2": sat(y * y), "prod": sat(x * y)}


def grid_window_sums(table: np.ndarray, k: int, stride: int) -> np.ndarray:
    h, w = table.shape[0] - 1, table.shape[1] - 1
    r_top, c_left = slice(0, h - k + 1, stride), slice(0, w - k + 1, stride)
    r_bot, c_right = slice(k, h + 1, stride), slice(k, w + 1, stride)
    return (table[r_bot, c_right] + table[r_top, c_left]) - (table[r_bot, c_left] + table[r_top, c_right])


TABLES = ("sum1", "sum2", "sq1", "sq2", "prod")


def box_window_sums(a: np.ndarray, b: np.ndarray, k: int, stride: int) -> np.ndarray:
    """The five exact int64 grids the integral engine forms: [5, gh, gw]."""
    iset = integral_set(a, b)
    return np.stack([grid_window_sums(iset[t], k, stride) for t in TABLES])


def sliding_sums(values: np.ndarray, weights: np.ndarray | None, k: int, stride: int) -> np.ndarray:
    """Direct windowed (weighted) sums: accumulate the k^2 shifted, strided slices."""
    h, w = values.shape
    gh, gw = h - k + 1, w - k + 1
    out = np.zeros(((gh - 1) // stride + 1, (gw - 1) // stride + 1), dtype=np.float64)
    for m in range(k):
        for n in range(k):
            view = values[m:m + gh:stride, n:n + gw:stride]
            out += view if weights is None else weights[m, n] * view
    return out


def moments_from_sums(s1, s2, q1, q2, p12, area: float):
    mu1 = s1 / area
    mu2 = s2 / area
    var1 = np.maximum(q1 / area - mu1 * mu1, 0.0)
    var2 = np.maximum(q2 / area - mu2 * mu2, 0.0)
    cov = p12 / area - mu1 * mu2
    return mu1, mu2, var1, var2, cov


def local_statistics(a: np.ndarray, b: np.ndarray, shape: str, k: int, stride: int = 1,
                     sigma: float | None = None, engine: str = "auto"):
    """(mu1, mu2, var1, var2, cov) float64 grids."""
    a, b = np.asarray(a), np.asarray(b)
    h, w = a.shape
    if k > h or k > w:
        raise ValueError("window larger than image")
    if engine == "auto":
        engine = "integral" if shape == "rect" else "naive"
    if engine == "integral" and shape != "rect":
        raise ValueError("integral engine needs a rect window")
    if engine == "integral":
        iset = integral_set(a, b)
        sums = [grid_window_sums(iset[t], k, stride).astype(np.float64) for t in TABLES]
        return moments_from_sums(*sums, area=float(k * k))
    fa = np.asarray(a, dtype=np.float64)
    fb = np.asarray(b, dtype=np.float64)
    weights = None if shape == "rect" else gaussian_kernel(sigma, k)
    sums = [sliding_sums(v, weights, k, stride) for v in (fa, fb, fa * fa, fb * fb, fa * fb)]
    return moments_from_sums(*sums, area=float(k * k) if shape == "rect" else 1.0)


def term_maps(mu1, mu2, var1, var2, cov, c1: float, c2: float):
    """(l, cs, q) float64 maps."""
    l_map = (2.0 * mu1 * mu2 + c1) / (mu1 * mu1 + mu2 * mu2 + c1)
    cs_map = (2.0 * cov + c2) / (var1 + var2 + c2)
    return l_map, cs_map, l_map * cs_map


def ssim_maps(a, b, shape: str = "rect", k: int = 11, stride: int = 1, sigma: float | None = None,
              bit_depth: int = 8, k1: float = 0.01, k2: float = 0.03, engine: str = "auto"):
    c1, c2 = constants(bit_depth, k1, k2)
    return term_maps(*local_statistics(a, b, shape, k, stride, sigma, engine), c1, c2)


def ssim_score(a, b, **window) -> float:
    return float(ssim_maps(a, b, **window)[2].mean())


def ssim_terms(a, b, **window) -> tuple[float, float, float]:
    """(mean q, mean l, mean cs) — the pipeline's (score/am, l_mean, cs_mean) record."""
    l_map, cs_map, q = ssim_maps(a, b, **window)
    return float(q.mean()), float(l_map.mean()), float(cs_map.mean())


# ---------------------------------------------------------------------------
# multiscale
# ---------------------------------------------------------------------------

def dyadic_downsample(values: np.ndarray) -> np.ndarray:
    arr = np.asarray(values, dtype=np.float64)
    h2, w2 = arr.shape[0] // 2, arr.shape[1] // 2
    arr = arr[: 2 * h2, : 2 * w2]
    return (arr[0::2, 0::2] + arr[0::2, 1::2] + arr[1::2, 0::2] + arr[1::2, 1::2]) / 4.0


def scale_scores(a, b, levels: int, **window) -> list[float]:
    k = window.get("k", 11)
    h, w = np.asarray(a).shape
    if min(h, w) // (1 << (levels - 1)) < k:
        raise ValueError("too many levels")
    cur_a, cur_b = a, b
    out = []
    for level in range(levels):
        if level > 0:
            cur_a, cur_b = dyadic_downsample(cur_a), dyadic_downsample(cur_b)
        _, cs_map, q = ssim_maps(cur_a, cur_b, **window)
        out.append(float((q if level == levels - 1 else cs_map).mean()))
    return out


def effective_exponents(aggregation: str, exponents) -> tuple:
    if aggregation in ("sum", "fast4"):
        total = sum(exponents)
        return tuple(e / total for e in exponents)
    return tuple(exponents)


def combine_scale_scores(scores, aggregation: str = "product", exponents=STANDARD_EXPONENTS) -> float:
    exps = effective_exponents(aggregation, exponents)
    if aggregation == "sum":
        return float(sum(e * s for e, s in zip(exps, scores)))
    out = 1.0
    for e, s in zip(exps, scores):
        out *= max(s, 0.0) ** e
    return float(out)


def msssim(a, b, levels: int = 5, aggregation: str = "product", exponents=None, **window) -> float:
    if exponents is None:
        exponents = STANDARD_EXPONENTS[:levels]
    return combine_scale_scores(scale_scores(a, b, levels, **window), aggregation, exponents)


# ---------------------------------------------------------------------------
# color + temporal
# ---------------------------------------------------------------------------

def channel_scores(ref_planes, dist_planes, **window) -> tuple[float, float, float]:
    """Per-channel mean SSIM, each plane at its own resolution (4:2:0 chroma stays 4:2:0)."""
    return tuple(ssim_score(a, b, **window) for a, b in zip(ref_planes, dist_planes))


def fixed_weight(scores, weights) -> float:
    return float(sum(w * s for w, s in zip(weights, scores)))


def channelwise(scores, alpha: float, beta: float) -> float:
    fy, fcb, fcr = scores
    return (fy + alpha * fcb + beta * fcr) / (1.0 + alpha + beta)


def pool_temporal_am(scores) -> float:
    return float(np.asarray(scores, dtype=np.float64).reshape(-1).mean())


# ---------------------------------------------------------------------------
# SSIM-3D rolling volumes (src/spatiotemporal.py:28-207)
# ---------------------------------------------------------------------------

class RollingSums:
    """Float64 rolling temporal sums exactly as the reference keeps them."""

    def __init__(self, kt: int, refresh_interval: int = 300):
        self.kt, self.refresh_interval = kt, refresh_interval
        self.buffer: list = []
        self.sums = None
        self.pushes = 0

    @staticmethod
    def _terms(a, b):
        return [a, b, a * a, b * b, a * b]

    def push(self, ref, dist):
        a = np.asarray(ref, dtype=np.float64)
        b = np.asarray(dist, dtype=np.float64)
        new = self._terms(a, b)
        if self.sums is None or self.kt == 1:
            self.sums = [t.copy() for t in new]
        elif len(self.buffer) == self.kt:
            old = self._terms(*self.buffer[0])
            for s, n_, o in zip(self.sums, new, old):
                s -= o
                s += n_
        else:
            for s, n_ in zip(self.sums, new):
                s += n_
        if len(self.buffer) == self.kt:
            self.buffer.pop(0)
        self.buffer.append((a, b))
        self.pushes += 1
        if self.refresh_interval and self.pushes % self.refresh_interval == 0:
            fresh = [np.zeros(a.shape) for _ in range(5)]
            for x, y in self.buffer:
                for s, t in zip(fresh, self._terms(x, y)):
                    s += t
            self.sums = fresh

    def stats(self, k: int, stride: int = 1):
        grids = [grid_window_sums(sat(s), k, stride) for s in self.sums]
        return moments_from_sums(*grids, area=float(k * k * len(self.buffer)))


def ssim3d_series(ref_frames, dist_frames, kt: int, k: int = 11, stride: int = 1, bit_depth: int = 8,
                  refresh_interval: int = 300) -> list:
    c1, c2 = constants(bit_depth)
    vol = RollingSums(kt, refresh_interval)
    out = []
    for a, b in zip(ref_frames, dist_frames):
        vol.push(a, b)
        out.append(float(term_maps(*vol.stats(k, stride), c1, c2)[2].mean()))
    return out


def msssim3d(ref_frames, dist_frames, kt: int, levels: int = 5, aggregation: str = "product", exponents=None,
             k: int = 11, stride: int = 1, bit_depth: int = 8) -> list:
    if exponents is None:
        exponents = STANDARD_EXPONENTS[:levels]
    c1, c2 = constants(bit_depth)
    vols = [RollingSums(kt) for _ in range(levels)]
    out = []
    for a, b in zip(ref_frames, dist_frames):
        cur_a, cur_b = a, b
        per = []
        for lv in range(levels):
            if lv:
                cur_a, cur_b = dyadic_downsample(cur_a), dyadic_downsample(cur_b)
            vols[lv].push(cur_a, cur_b)
            _, cs_map, q = term_maps(*vols[lv].stats(k, stride), c1, c2)
            per.append(float((q if lv == levels - 1 else cs_map).mean()))
        out.append(combine_scale_scores(per, aggregation, exponents))
    return out


# ---------------------------------------------------------------------------
# resolution adaptation (src/adaptation.py:23-110)
# ---------------------------------------------------------------------------

def round_half_away(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def scale_factor(kind: str, width: int, height: int, rounding: str = "round", d_over_h: float = 3.0,
                 distance: float | None = None, theta_h: float = 40.0, theta_w: float = 50.0) -> int:
    """Integer factor of a scale policy: none / legacy (256-line rule) / dh / sast."""
    if kind == "none":
        return 1
    if kind in ("legacy", "dh"):
        ratio = min(width, height) / 256.0
        if kind == "dh":
            ratio = ratio * (3.0 / d_over_h)
        r = math.ceil(ratio) if rounding == "ceil" else round_half_away(ratio)
        return max(1, r)
    denom = 4.0 * math.tan(math.radians(theta_h) / 2.0) * math.tan(math.radians(theta_w) / 2.0)
    z = max(1.0, math.sqrt((height / distance) * (width / distance) / denom))
    return max(1, round_half_away(z))


def box_downsample(values: np.ndarray, factor: int) -> np.ndarray:
    """Block means over factor x factor blocks; trailing blocks average their real size."""
    if factor == 1:
        return values
    x = np.asarray(values, dtype=np.float64)
    h, w = x.shape
    rows, cols = np.arange(0, h, factor), np.arange(0, w, factor)
    block = np.add.reduceat(np.add.reduceat(x, rows, axis=0), cols, axis=1)
    counts = np.outer(np.minimum(rows + factor, h) - rows, np.minimum(cols + factor, w) - cols)
    return block / counts


# ---------------------------------------------------------------------------
# spatial pooling (src/pooling.py:157-243)
# ---------------------------------------------------------------------------

def pool_spatial(values, kind: str, p: float = 1.0, o: float = 1.0, a: float = 0.0, b: float = 0.0,
                 ps: float = 6.0, rs: float = 1.0, ref_luma=None) -> float:
    v = np.asarray(values, dtype=np.float64).reshape(-1)
    if v.size == 0:
        raise ValueError("empty map")
    if kind == "am":
        return float(v.mean())
    if kind == "cov":
        m = v.mean()
        if m == 0.0:
            raise ZeroDivisionError("zero-mean map")
        return float(v.std() / m)
    if kind == "md":
        spread = (np.abs(v - v.mean()) ** p).mean()
        return float((spread ** (1.0 / p)) ** o)
    if kind == "fns":
        lo, mid, hi = np.percentile(v, [25.0, 50.0, 75.0])
        return float((v.min() + lo + mid + hi + v.max()) / 5.0)
    if kind == "dw":
        wt = (1.0 - v) ** p
        tot = wt.sum()
        return float(v.mean()) if tot == 0.0 else float((wt * v).sum() / tot)
    if kind == "mink":
        return float(((1.0 - v) ** p).mean())
    if kind == "pp":
        if ps <= 0.0 or rs == 1.0:
            return float(v.mean())
        cut = np.percentile(v, ps)
        return float(np.where(v <= cut, v / rs, v).mean())
    if kind == "lw":
        mu = np.asarray(ref_luma, dtype=np.float64).reshape(-1)
        wt = (mu >= a).astype(np.float64) if b == 0.0 else np.clip((mu - a) / b, 0.0, 1.0)
        return float((wt * v).mean())
    raise ValueError(f"unknown pooler {kind!r}")


def luma_frame_record(ref, dist, shape: str = "rect", k: int = 11, stride: int = 1, sigma: float | None = None,
                      bit_depth: int = 8, engine: str = "auto", factor: int = 1, pool: str = "am",
                      **pool_params) -> tuple[float, float, float, float]:
    """(score, am, l_mean, cs_mean) of one luma pair: downsample, statistics, maps, pooling."""
    x = box_downsample(np.asarray(ref), factor)
    y = box_downsample(np.asarray(dist), factor)
    stats = local_statistics(x, y, shape, k, stride, sigma, engine)
    c1, c2 = constants(bit_depth)
    l_map, cs_map, q = term_maps(*stats, c1, c2)
    score = pool_spatial(q, pool, ref_luma=stats[0], **pool_params)
    return score, float(q.mean()), float(l_map.mean()), float(cs_map.mean())


# ---------------------------------------------------------------------------
# colorimetric models (src/color.py:27-371)
# ---------------------------------------------------------------------------

KR, KG, KB = 0.213, 0.715, 0.072
CB_SCALE, CR_SCALE = 0.539, 0.635
RGB_TO_XYZ = np.array([[0.4124564, 0.3575761, 0.1804375],
                       [0.2126729, 0.7151522, 0.0721750],
                       [0.0193339, 0.1191920, 0.9503041]])
D65 = (0.95047, 1.0, 1.08883)
XYZ_TO_Q = np.array([[0.279, 0.72, -0.107], [-0.449, 0.29, -0.077], [0.086, -0.59, 0.501]])
Q_TO_XYZ = np.array([[0.6204, -1.8704, -0.1553], [1.3661, 0.9316, 0.4339], [1.5013, 1.4176, 2.5331]])
DELTA_E_FULL_MASK = 45.0


def _f64(chans):
    return [np.asarray(c, dtype=np.float64) for c in chans]


def upsample420(chans, h: int, w: int):
    """Nearest-neighbour chroma upsampling to the luma grid."""
    y, cb, cr = chans
    return [y] + [np.repeat(np.repeat(c, 2, axis=0), 2, axis=1)[:h, :w] for c in (cb, cr)]


def rgb_to_ycbcr(chans, peak: float):
    r, g, b = _f64(chans)
    y = KR * r + KG * g + KB * b
    half = peak / 2.0
    return [y, CB_SCALE * (b - y) + half, CR_SCALE * (r - y) + half]


def ycbcr_to_rgb(chans, peak: float):
    """Inverse BT.709 of 4:4:4 channels, clamped to [0, peak]."""
    y, cb, cr = _f64(chans)
    half = peak / 2.0
    b = (cb - half) / CB_SCALE + y
    r = (cr - half) / CR_SCALE + y
    g = (y - KR * r - KB * b) / KG
    return [np.clip(c, 0.0, peak) for c in (r, g, b)]


def luma_rgb(chans):
    r, g, b = _f64(chans)
    return KR * r + KG * g + KB * b


def hue(chans, peak: float):
    """HSV hue scaled to [0, peak]; achromatic pixels 0."""
    r, g, b = _f64(chans)
    hi = np.maximum(np.maximum(r, g), b)
    lo = np.minimum(np.minimum(r, g), b)
    d = hi - lo
    safe = np.where(d == 0.0, 1.0, d)
    h = np.where(d == 0.0, 0.0,
                 np.where(hi == r, np.mod((g - b) / safe, 6.0),
                          np.where(hi == g, (b - r) / safe + 2.0, (r - g) / safe + 4.0)))
    h = h * 60.0
    return h / 360.0 * peak


def smooth_reflect(values, sigma: float = 2.0, k: int = 13):
    """Separable Gaussian, reflect padding, same-size output."""
    g = gaussian_kernel(sigma, k)[(k - 1) // 2]
    g = g / g.sum()
    pad = (k - 1) // 2
    v = np.pad(values, ((pad, pad), (0, 0)), mode="reflect")
    v = sum(g[m] * v[m:m + values.shape[0], :] for m in range(k))
    v = np.pad(v, ((0, 0), (pad, pad)), mode="reflect")
    return sum(g[n] * v[:, n:n + values.shape[1]] for n in range(k))


def rgb_to_lab(chans, peak: float, smooth: bool = False):
    rgb = np.stack([np.asarray(c, dtype=np.float64) / peak for c in chans])
    xyz = RGB_TO_XYZ @ rgb.reshape(3, -1)
    if smooth:
        q = (XYZ_TO_Q @ xyz).reshape(3, *rgb.shape[1:])
        q = np.stack([q[0], smooth_reflect(q[1]), smooth_reflect(q[2])])
        xyz = Q_TO_XYZ @ q.reshape(3, -1)
    x, y, z = (c.reshape(rgb.shape[1:]) for c in xyz)

    def f(t):
        d = 6.0 / 29.0
        return np.where(t > d ** 3, np.cbrt(t), t / (3 * d * d) + 4.0 / 29.0)

    fx, fy, fz = f(x / D65[0]), f(y / D65[1]), f(z / D65[2])
    return [116.0 * fy - 16.0, 500.0 * (fx - fy), 200.0 * (fy - fz)]


def delta_e(rgb1, rgb2, peak: float, smooth: bool = True):
    l1, l2 = rgb_to_lab(rgb1, peak, smooth), rgb_to_lab(rgb2, peak, smooth)
    return np.sqrt(sum((a - b) ** 2 for a, b in zip(l1, l2)))


def qssim(emb1, emb2, k: int, stride: int, peak: float, k1: float = 0.01, k2: float = 0.03) -> float:
    """Quaternion SSIM of two 3-channel embeddings (pure quaternions on i, j, k)."""
    r1, g1, b1 = _f64(emb1)
    r2, g2, b2 = _f64(emb2)
    c1, c2 = (k1 * peak) ** 2, (k2 * peak) ** 2
    kern = np.full((k, k), 1.0 / (k * k))

    def wm(x):
        return sliding_sums(x, kern, k, stride)

    m1 = [wm(r1), wm(g1), wm(b1)]
    m2 = [wm(r2), wm(g2), wm(b2)]
    e_dot = wm(r1 * r2 + g1 * g2 + b1 * b2)
    e_i = wm(-(g1 * b2 - b1 * g2))
    e_j = wm(-(b1 * r2 - r1 * b2))
    e_k = wm(-(r1 * g2 - g1 * r2))
    e_sq1 = wm(r1 * r1 + g1 * g1 + b1 * b1)
    e_sq2 = wm(r2 * r2 + g2 * g2 + b2 * b2)
    mdot = m1[0] * m2[0] + m1[1] * m2[1] + m1[2] * m2[2]
    mi = -(m1[1] * m2[2] - m1[2] * m2[1])
    mj = -(m1[2] * m2[0] - m1[0] * m2[2])
    mk = -(m1[0] * m2[1] - m1[1] * m2[0])
    n1 = m1[0] ** 2 + m1[1] ** 2 + m1[2] ** 2
    n2 = m2[0] ** 2 + m2[1] ** 2 + m2[2] ** 2
    num1 = np.sqrt((2.0 * mdot + c1) ** 2 + (2.0 * mi) ** 2 + (2.0 * mj) ** 2 + (2.0 * mk) ** 2)
    num2 = np.sqrt((2.0 * (e_dot - mdot) + c2) ** 2 + (2.0 * (e_i - mi)) ** 2 + (2.0 * (e_j - mj)) ** 2
                   + (2.0 * (e_k - mk)) ** 2)
    den1 = n1 + n2 + c1
    den2 = (e_sq1 - n1) + (e_sq2 - n2) + c2
    return float(((num1 / den1) * (num2 / den2)).mean())


def qssim_embedding(chans, space: str, peak: float, ycc: bool = False, h: int = 0, w: int = 0):
    """Embedding channels: rgb as is, BT.709 YCbCr (converted from RGB or upsampled 4:2:0), Lab * peak/100."""
    if ycc:
        chans = upsample420(chans, h, w)
        if space == "ycbcr":
            return _f64(chans)
        chans = ycbcr_to_rgb(chans, peak)
    if space == "rgb":
        return _f64(chans)
    if space == "ycbcr":
        return rgb_to_ycbcr(chans, peak)
    return [c * (peak / 100.0) for c in rgb_to_lab(chans, peak)]


def cmssim(rgb1, rgb2, peak: float, bit_depth: int, **window) -> float:
    """Luma SSIM map weighted by clamp(1 - dE/45, 0, 1) sampled at window centres."""
    _, _, q = ssim_maps(luma_rgb(rgb1), luma_rgb(rgb2), bit_depth=bit_depth, **window)
    wgt = np.clip(1.0 - delta_e(rgb1, rgb2, peak, True) / DELTA_E_FULL_MASK, 0.0, 1.0)
    k, s = window["k"], window.get("stride", 1)
    c = (k - 1) // 2
    rows = np.arange(q.shape[0]) * s + c
    cols = np.arange(q.shape[1]) * s + c
    return float((q * wgt[np.ix_(rows, cols)]).mean())


def hssim(rgb1, rgb2, peak: float, bit_depth: int, **window) -> float:
    luma = ssim_maps(luma_rgb(rgb1), luma_rgb(rgb2), bit_depth=bit_depth, **window)[2].mean()
    hue_s = ssim_maps(hue(rgb1, peak), hue(rgb2, peak), bit_depth=bit_depth, **window)[2].mean()
    return float((luma + 0.2 * hue_s) / 1.2)
