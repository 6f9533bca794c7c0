"""Exception hierarchy of the engine, mirroring ssimkit's (src/errors.py).

The drop-in promise is that callers catching the reference's exception
classes keep working, so every class below has the reference's name, base
classes and meaning.  Native (C-ABI) error codes are translated onto these in
``_native.raise_for``.
"""

from __future__ import annotations


class SsimkitError(Exception):
    """Root of every error raised by the engine (src/errors.py:9-10)."""


class ValidationError(SsimkitError, ValueError):
    """An argument breaks a construction invariant (src/errors.py:13-14)."""


# pair / frame checks
class DimensionMismatch(SsimkitError):
    """Reference and distorted geometry differ (src/errors.py:19)."""


class BitDepthMismatch(SsimkitError):
    """Reference and distorted bit depths differ (src/errors.py:23)."""


class WrongSpace(SsimkitError):
    """Frame is tagged with a color space the operation cannot take."""


# windows / statistics
class NonPositiveSigma(SsimkitError, ValueError):
    """Gaussian sigma <= 0."""


class EngineShapeMismatch(SsimkitError):
    """``engine='integral'`` asked for a non-rectangular window (src/errors.py:63)."""


class WindowLargerThanImage(SsimkitError):
    """Window does not fit the plane (src/errors.py:67)."""


class WindowOutOfBounds(SsimkitError):
    """A single-window query leaves the valid region."""


class GaussianNotSupported3D(SsimkitError):
    """Spatio-temporal statistics take rectangular windows only."""


# multiscale
class TooSmall(SsimkitError):
    """Plane too small for the operation (src/errors.py:81)."""


class TooManyLevels(SsimkitError):
    """Coarsest requested scale cannot hold one window (src/errors.py:85)."""


# pooling
class EmptyMap(SsimkitError):
    """Nothing to pool in a quality map (src/errors.py:91)."""


class EmptySeries(SsimkitError):
    """Nothing to pool in a score series."""


class ZeroMeanCoV(SsimkitError):
    """Coefficient of variation of a zero-mean input."""


class MissingLumaForLW(SsimkitError):
    """Luminance-weighted pooling without a co-registered mean-luma map."""


class DegenerateWeights(SsimkitError):
    """Channel weights with a zero normaliser."""


class DegenerateData(SsimkitError):
    """Data cannot support the requested statistic."""


class EngineUnavailable(SsimkitError, RuntimeError):
    """The CUDA engine (libssimk.so on a B200) is missing: there is no CPU fallback."""


# media ingest (src/errors.py, media section)
class BadMagic(SsimkitError):
    """Stream does not start with the expected magic token."""


class BadHeader(SsimkitError):
    """Header could not be parsed."""


class UnsupportedChroma(SsimkitError):
    """Chroma subsampling tag is not supported."""


class TruncatedFrame(SsimkitError):
    """Frame payload is shorter than the declared plane sizes."""


class SizeNotMultiple(SsimkitError):
    """Raw file size is not a whole multiple of the frame size."""


class UnsupportedMaxval(SsimkitError):
    """PNM maxval is zero or exceeds the 16-bit range."""


class LengthMismatch(SsimkitError):
    """Paired sequences differ in length."""


# The two classes below belong to reference subsystems outside the hot path (the scaled-SSIM
# histogram matcher, the evaluation harness: SURVEY.md §8 OUT); they complete the exception
# hierarchy (src/errors.py:113-128) so code catching them still imports.
class NoReferenceYet(SsimkitError):
    """Histogram matcher was asked to predict before any reference map."""


class TooFew(SsimkitError):
    """Not enough samples for the requested statistic."""
