"""Media ingest straight into the scoring batches (ssimkit src/media.py:94-212).

Y4M (8-bit; YUV4MPEG2 header, FRAME markers) and headerless planar YUV
(8-bit, or little-endian 16-bit) are memory-mapped; frame offsets are found
once, and each frame's planes are zero-copy ``numpy`` views into the mapping,
so batches are filled by one copy per plane into the pinned staging buffers of
``SequenceScorer`` (no per-frame parsing on the hot loop).  Header grammar,
chroma tags and error classes follow the reference readers.
"""

from __future__ import annotations

import contextlib

import os
from dataclasses import dataclass
from typing import Iterator, Optional, Sequence

import numpy as np

from .errors import (
    BadHeader,
    BadMagic,
    SizeNotMultiple,
    TruncatedFrame,
    UnsupportedChroma,
    UnsupportedMaxval,
    ValidationError,
)
from .planes import CHROMA_420, CHROMA_444, SPACE_RGB, SPACE_YCBCR, ColorFrame, LumaPlane

Y4M_MAGIC = b"YUV4MPEG2"
_Y4M_CHROMA = {"420": CHROMA_420, "420jpeg": CHROMA_420, "420mpeg2": CHROMA_420, "444": CHROMA_444, "mono": "mono"}


@dataclass(frozen=True)
class StreamHeader:
    width: int
    height: int
    frame_rate: tuple
    chroma: str  # "420" | "444" | "mono"
    bit_depth: int = 8

    @property
    def fps(self) -> float:
        return self.frame_rate[0] / self.frame_rate[1]

    def plane_shapes(self) -> list:
        if self.chroma == "mono":
            return [(self.height, self.width)]
        if self.chroma == CHROMA_420:
            c = ((self.height + 1) // 2, (self.width + 1) // 2)
        else:
            c = (self.height, self.width)
        return [(self.height, self.width), c, c]

    @property
    def sample_dtype(self):
        return np.dtype(np.uint8) if self.bit_depth <= 8 else np.dtype("<u2")

    def frame_bytes(self) -> int:
        es = self.sample_dtype.itemsize
        return sum(h * w * es for h, w in self.plane_shapes())


class FrameSource:
    """Memory-mapped frames of one stream; ``planes(i)`` gives views into the file."""

    def __init__(self, path, header: StreamHeader, offsets: Sequence[int]):
        self.path = str(path)
        self.header = header
        self._offsets = list(offsets)
        # np.memmap keeps the mapping alive for as long as any returned plane view exists; a
        # private (copy-on-write) mapping, because the driver page-locks private mappings
        # (pin) but refuses shared file mappings.  Nothing ever writes through it.
        size = os.path.getsize(self.path)
        self._buf = np.memmap(self.path, dtype=np.uint8, mode="c") if size else np.zeros(0, np.uint8)

    def __len__(self) -> int:
        return len(self._offsets)

    def planes(self, i: int) -> tuple:
        off = self._offsets[i]
        es = self.header.sample_dtype.itemsize
        out = []
        for h, w in self.header.plane_shapes():
            n = h * w * es
            out.append(self._buf[off:off + n].view(self.header.sample_dtype).reshape(h, w))
            off += n
        return tuple(out)

    def luma(self) -> Iterator[np.ndarray]:
        for i in range(len(self)):
            yield self.planes(i)[0]

    def frames(self) -> Iterator[tuple]:
        for i in range(len(self)):
            yield self.planes(i)

    @property
    def pinned(self) -> bool:
        return getattr(self, "_pinned", False)

    def pin(self) -> bool:
        """Page-lock the mapping (``ssk_host_register``) so the scorer DMAs frame
        planes straight from the page cache with no staging copy.  False if the driver
        refuses (the scorer then packs through its pinned buffers as usual)."""
        if self.pinned or self._buf.size == 0:
            return self.pinned
        from . import _native as nat

        nat.require_device()
        self._pinned = nat.lib().ssk_host_register(self._buf.ctypes.data, self._buf.nbytes, 0) == 0
        return self._pinned

    def unpin(self) -> None:
        if self.pinned:
            from . import _native as nat

            nat.lib().ssk_host_unregister(self._buf.ctypes.data)
            self._pinned = False

    def close(self) -> None:
        """Drop this source's reference to the mapping (views handed out stay valid)."""
        self.unpin()
        self._buf = np.zeros(0, np.uint8)


def _parse_y4m_header(line: str) -> StreamHeader:
    width = height = None
    rate = (30, 1)
    chroma = CHROMA_420
    for tok in line.split(" "):
        if not tok:
            continue
        tag, val = tok[0], tok[1:]
        if tag == "W":
            width = int(val)
        elif tag == "H":
            height = int(val)
        elif tag == "F":
            num, _, den = val.partition(":")
            rate = (int(num), int(den or "1"))
        elif tag == "C":
            if val not in _Y4M_CHROMA:
                raise UnsupportedChroma(f"chroma tag C{val} is not supported")
            chroma = _Y4M_CHROMA[val]
        elif tag in ("I", "A", "X"):
            continue
        else:
            raise BadHeader(f"unknown header token {tok!r}")
    if not width or not height or width <= 0 or height <= 0:
        raise BadHeader(f"header lacks valid dimensions: {line!r}")
    return StreamHeader(width, height, rate, chroma, 8)


def open_y4m(path) -> FrameSource:
    """Index a YUV4MPEG2 file (src/media.py:94-175): one pass over the FRAME markers."""
    with open(path, "rb") as fh:
        data = fh.read()
    if not data.startswith(Y4M_MAGIC):
        raise BadMagic(f"{path}: not a YUV4MPEG2 stream")
    eol = data.find(b"\n")
    if eol < 0 or eol > 512:
        raise BadHeader("unterminated header line")
    header = _parse_y4m_header(data[len(Y4M_MAGIC):eol].decode("ascii", "replace"))
    fbytes = header.frame_bytes()
    pos, offsets = eol + 1, []
    while pos < len(data):
        nl = data.find(b"\n", pos, pos + 512)
        if nl < 0:
            raise BadHeader("unterminated FRAME marker")
        if not data[pos:nl].startswith(b"FRAME"):
            raise BadHeader(f"expected FRAME marker, got {data[pos:pos + 20]!r}")
        start = nl + 1
        if start + fbytes > len(data):
            raise TruncatedFrame(f"frame needs {fbytes} bytes, stream had {len(data) - start}")
        offsets.append(start)
        pos = start + fbytes
    return FrameSource(path, header, offsets)


def open_raw(path, width: int, height: int, bit_depth: int = 8, chroma: str = CHROMA_420,
             frame_rate=(30, 1)) -> FrameSource:
    """Index a headerless planar YUV file (src/media.py:178-212)."""
    if width <= 0 or height <= 0:
        raise ValidationError("dimensions must be positive")
    if chroma == "400":
        chroma = "mono"
    if chroma not in (CHROMA_420, CHROMA_444, "mono"):
        raise UnsupportedChroma(f"chroma {chroma!r} not supported for raw input")
    header = StreamHeader(width, height, tuple(frame_rate), chroma, bit_depth)
    fbytes = header.frame_bytes()
    size = os.path.getsize(path)
    if size == 0 or size % fbytes != 0:
        raise SizeNotMultiple(f"{path}: {size} bytes is not a whole number of {fbytes}-byte frames")
    return FrameSource(path, header, [i * fbytes for i in range(size // fbytes)])


def _frame_planes(fr) -> tuple:
    """Planes of a frame given as LumaPlane / ColorFrame (reference types) or arrays."""
    if isinstance(fr, LumaPlane):
        return (fr.samples,)
    if isinstance(fr, ColorFrame):
        return tuple(fr.channels)
    return tuple(fr) if isinstance(fr, (tuple, list)) else (fr,)


def write_y4m(path, frames, width, height: Optional[int] = None, chroma: str = CHROMA_420,
              frame_rate=(30, 1)) -> None:
    """Write 8-bit frames as YUV4MPEG2: ``write_y4m(path, frames, header)`` as in the
    reference (src/media.py:272-281), or with explicit width / height / chroma."""
    if isinstance(width, StreamHeader):
        hd = width
        width, height, chroma, frame_rate = hd.width, hd.height, hd.chroma, hd.frame_rate
    tag = {CHROMA_420: "420jpeg", CHROMA_444: "444", "mono": "mono"}[chroma]
    with open(path, "wb") as fh:
        fh.write(Y4M_MAGIC + f" W{width} H{height} F{frame_rate[0]}:{frame_rate[1]} C{tag}\n".encode())
        for fr in frames:
            fh.write(b"FRAME\n")
            for p in _frame_planes(fr):
                fh.write(np.ascontiguousarray(p, dtype=np.uint8).tobytes())


def write_planar_raw(path, frames, bit_depth: int = 8) -> None:
    """Write frames as headerless planar YUV (little-endian for > 8 bits)."""
    dt = np.uint8 if bit_depth <= 8 else np.dtype("<u2")
    with open(path, "wb") as fh:
        for fr in frames:
            for p in _frame_planes(fr):
                fh.write(np.ascontiguousarray(p, dtype=dt).tobytes())


# ---------------------------------------------------------------------------
# reference-named readers (src/media.py:58-237) over the memory-mapped sources
# ---------------------------------------------------------------------------

class VideoStream:
    """Stream header plus frames (src/media.py:58-70); iterating yields LumaPlane for mono
    streams and YCbCr ColorFrame otherwise, each a zero-copy view of the mapping."""

    def __init__(self, source: FrameSource):
        self.source = source
        self.header = source.header

    def __len__(self) -> int:
        return len(self.source)

    def frame(self, i: int):
        planes = self.source.planes(i)
        bd = self.header.bit_depth
        if self.header.chroma == "mono":
            return LumaPlane(planes[0], bd)
        return ColorFrame(planes, SPACE_YCBCR, self.header.chroma, bd)

    def __iter__(self):
        for i in range(len(self.source)):
            yield self.frame(i)

    def luma_frames(self):
        for y in self.source.luma():
            yield LumaPlane(y, self.header.bit_depth)


def read_y4m(path) -> VideoStream:
    """Open a YUV4MPEG2 file (src/media.py:94-118)."""
    return VideoStream(open_y4m(path))


def read_planar_raw(path, width: int, height: int, bit_depth: int = 8, chroma: str = CHROMA_420,
                    frame_rate=(30, 1)) -> VideoStream:
    """Open a headerless planar YUV file; dimensions from the caller (src/media.py:178-212)."""
    return VideoStream(open_raw(path, width, height, bit_depth, chroma, frame_rate))


def read_pnm(path):
    """Binary PNM (src/media.py:215-269): P5 -> LumaPlane, P6 -> RGB ColorFrame; 16-bit big-endian."""
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:2] not in (b"P5", b"P6"):
        raise BadHeader(f"{path}: not a binary P5/P6 PNM file")
    kind = data[:2].decode()
    fields: list = []
    i = 2
    while len(fields) < 3:
        if i >= len(data):
            raise BadHeader(f"{path}: truncated PNM header")
        c = data[i:i + 1]
        if c == b"#":
            while i < len(data) and data[i:i + 1] != b"\n":
                i += 1
        elif c.isspace():
            i += 1
        elif c.isdigit():
            j = i
            while j < len(data) and data[j:j + 1].isdigit():
                j += 1
            fields.append(int(data[i:j]))
            i = j
        else:
            raise BadHeader(f"{path}: unexpected byte {c!r} in PNM header")
    i += 1  # the single whitespace byte after maxval
    width, height, maxval = fields
    if width <= 0 or height <= 0:
        raise BadHeader(f"{path}: bad dimensions {width}x{height}")
    if maxval <= 0 or maxval > 65535:
        raise UnsupportedMaxval(f"maxval {maxval} outside (0, 65535]")
    bd = 8 if maxval <= 255 else 16
    dt = np.dtype(np.uint8) if bd == 8 else np.dtype(">u2")
    nch = 1 if kind == "P5" else 3
    count = width * height * nch
    payload = np.frombuffer(data, dtype=dt, count=min(count, (len(data) - i) // dt.itemsize), offset=i)
    if payload.size < count:
        raise TruncatedFrame(f"{path}: expected {count} samples, found {payload.size}")
    if kind == "P5":
        return LumaPlane(payload.reshape(height, width), bd)
    rgb = payload.reshape(height, width, 3)
    return ColorFrame((rgb[:, :, 0], rgb[:, :, 1], rgb[:, :, 2]), SPACE_RGB, CHROMA_444, bd)


def open_stream(path, width: Optional[int] = None, height: Optional[int] = None, bit_depth: int = 8,
                chroma: str = CHROMA_420):
    """Any supported media file as a stream (src/pipeline.py:118-141); images -> 1-frame lists."""
    ext = os.path.splitext(str(path))[1].lower()
    if ext == ".y4m":
        return read_y4m(path)
    if ext in (".pnm", ".pgm", ".ppm"):
        return [read_pnm(path)]
    if width is None or height is None:
        raise ValidationError(f"{path}: raw planar input needs explicit --width and --height")
    return read_planar_raw(path, width, height, bit_depth, chroma)


# ---------------------------------------------------------------------------
# report writer (src/media.py:310-372): deterministic, byte-for-byte output
# ---------------------------------------------------------------------------

def format_float(x: float) -> str:
    """9 significant digits, trailing zeros kept (1 -> 1.00000000)."""
    return format(float(x), "#.9g")


def _cell_csv(v) -> str:
    if v is None:
        return ""
    if isinstance(v, bool):
        return str(v).lower()
    if isinstance(v, float):
        return "" if v != v else format_float(v)
    return str(v)


def _cell_json(v) -> str:
    import json

    if v is None:
        return "null"
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        return "null" if v != v else format_float(v)
    if isinstance(v, int):
        return str(v)
    return json.dumps(str(v))


def write_report(records, fmt: str = "jsonl", fields=None) -> bytes:
    """Serialise per-frame records with a fixed field order (jsonl or csv)."""
    import json

    if fmt not in ("jsonl", "csv"):
        raise ValidationError(f"unknown report format {fmt!r}")
    if fields is None:
        if not records:
            raise ValidationError("empty record list needs an explicit field list")
        fields = list(records[0].keys())
    for i, rec in enumerate(records):
        if set(rec.keys()) != set(fields):
            raise ValidationError(f"record {i} does not match the report schema {list(fields)}")
    if fmt == "csv":
        lines = [",".join(fields)] + [",".join(_cell_csv(r[f]) for f in fields) for r in records]
    else:
        lines = ["{" + ", ".join(f"{json.dumps(f)}: {_cell_json(r[f])}" for f in fields) + "}" for r in records]
    return ("\n".join(lines) + "\n").encode()


def score_files(ref: FrameSource, dist: FrameSource, config=None, batch_frames: int = 16,
                color_weights: Optional[Sequence[float]] = None):
    """Score two indexed streams frame by frame on the GPU (the reference's run_score frame loop,
    src/pipeline.py:275-366, for the luma / multiscale / fixed-weight color models)."""
    from .options import SsimConfig
    from .video import SequenceScorer

    config = config or SsimConfig()
    if (ref.header.width, ref.header.height) != (dist.header.width, dist.header.height):
        from .errors import DimensionMismatch

        raise DimensionMismatch("reference and distorted streams differ in size")
    if len(ref) != len(dist):
        raise ValidationError(f"streams differ in length: {len(ref)} vs {len(dist)} frames")
    cfg = config.for_bit_depth(ref.header.bit_depth)
    scorer = SequenceScorer(cfg, batch_frames, color_weights)
    with pinned_pair(ref, dist) as direct:  # page-locked mappings: planes DMA'd with no host copy
        if color_weights is not None:
            return scorer.score(ref.frames(), dist.frames(), direct=direct)
        return scorer.score(ref.luma(), dist.luma(), direct=direct)


@contextlib.contextmanager
def pinned_pair(ref: FrameSource, dist: FrameSource):
    """Page-lock both mappings for the duration of the block (yields whether both are pinned);
    always unpins what it pinned, also when the second pin fails or scoring raises."""
    pinned = []
    try:
        for src in (ref, dist):
            if src.pinned:
                continue
            if not src.pin():
                break
            pinned.append(src)
        yield ref.pinned and dist.pinned
    finally:
        for src in pinned:
            src.unpin()
