"""Image validation and the declared intensity range.

Restates the boundary semantics of `/root/reference/pkg/src/fastbilateral/image.py:19-66`
(`RangeSpec`, `RANGE_8BIT`, `as_image`, `validate_range`, `center`,
`uncenter`).  File I/O (PGM/PNG) is out of scope for this hot-path build.

The GPU path does NOT call `as_image`/`validate_range` on large inputs: the
channel-generation kernel checks finiteness and range while it reads the image
(first offending pixel in row-major order, identical to `np.argwhere(bad)[0]`),
and `_native.py` raises the same exceptions with the same messages.
These host versions are kept for API parity and for the small-input paths.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ParameterError, RangeViolationError


@dataclass(frozen=True)
class RangeSpec:
    """Samples are declared to lie in [center - half_range, center + half_range]."""

    half_range: float
    center: float = 0.0

    def __post_init__(self):
        if not self.half_range > 0:
            raise ParameterError(f"half_range must be positive, got {self.half_range}")

    @property
    def lo(self) -> float:
        return self.center - self.half_range

    @property
    def hi(self) -> float:
        return self.center + self.half_range


#: 8-bit data: [0, 255] is centred by 128 into [-128, 127].
RANGE_8BIT = RangeSpec(half_range=128.0, center=128.0)


def range_message(value, row, col, lo, hi) -> str:
    return f"sample {value} at pixel (row={row}, col={col}) outside [{lo}, {hi}]"


def as_image(arr) -> np.ndarray:
    """Return `arr` as a validated non-empty, finite, 2-D float64 array."""
    img = np.asarray(arr, dtype=np.float64)
    if img.ndim != 2 or img.size == 0:
        raise ParameterError(f"image must be a non-empty 2-D array, got shape {img.shape}")
    if not np.isfinite(img).all():
        raise ParameterError("image contains non-finite samples")
    return img


def validate_range(img: np.ndarray, spec: RangeSpec) -> None:
    """Raise `RangeViolationError` naming the first (row-major) out-of-range sample."""
    lo, hi = spec.lo, spec.hi
    outside = np.flatnonzero(((img < lo) | (img > hi)).ravel())
    if outside.size:
        row, col = divmod(int(outside[0]), img.shape[1])
        raise RangeViolationError(range_message(img[row, col], row, col, lo, hi))


def center(img, spec: RangeSpec) -> np.ndarray:
    img = as_image(img)
    validate_range(img, spec)
    return img - spec.center


def uncenter(img, spec: RangeSpec) -> np.ndarray:
    return as_image(img) + spec.center
