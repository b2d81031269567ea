"""Image validation and the declared intensity range.

Restates the boundary semantics of `/root/reference/pkg/src/fastbilateral/image.py:19-66`
(`RangeSpec`, `RANGE_8BIT`, `as_image`, `validate_range`, `center`,
`uncenter`) and the file I/O of `image.py:69-129` (`load_pgm`, `save_pgm`, `load_image`,
`save_image`; binary P5 PGM with maxval 255, 8-bit grayscale PNG through Pillow).

File I/O keeps the raster in its 8-bit form on the filter path:
`read_raster` returns the file's bytes as a uint8 view (no float64 promotion on the host), the
filter kernels read uint8 directly, and `gpa_filter(..., out_dtype=np.uint8)` quantises in kernel
2's epilogue exactly as `save_pgm` does, so `write_raster` writes the returned bytes as they are.
A PGM -> filter -> PGM round trip therefore moves 1 byte per pixel each way over PCIe instead of
8.  `load_pgm` / `load_image` / `save_pgm` / `save_image` keep the reference's float64 contract.

The GPU path does NOT call `as_image`/`validate_range` on large inputs: the
channel-generation kernel checks finiteness and range while it reads the image
(first offending pixel in row-major order, identical to `np.argwhere(bad)[0]`),
and `_native.py` raises the same exceptions with the same messages.
These host versions are kept for API parity and for the small-input paths.
"""

from __future__ import annotations

import re
from dataclasses import dataclass
from pathlib import Path

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


# ---------------------------------------------------------------------------- file I/O
_PGM_TOKEN = re.compile(rb"\s*(?:#[^\n]*\n\s*)*(\d+)")


def _parse_pgm(path, data: bytes) -> np.ndarray:
    """uint8 (H, W) view of a binary P5 PGM's raster (header grammar of image.py:73-93)."""
    if not data.startswith(b"P5"):
        raise ValueError(f"{path}: not a binary PGM (missing P5 magic)")
    fields, pos = [], 2
    for _ in range(3):  # width, height, maxval; '#' comment lines may sit between them
        m = _PGM_TOKEN.match(data, pos)
        if m is None:
            raise ValueError(f"{path}: malformed PGM header")
        fields.append(int(m.group(1)))
        pos = m.end()
    width, height, maxval = fields
    if maxval != 255:
        raise ValueError(f"{path}: only maxval 255 supported, got {maxval}")
    pos += 1  # the single whitespace byte that ends the header
    if len(data) - pos < width * height:
        raise ValueError(f"{path}: truncated raster")
    return np.frombuffer(data, dtype=np.uint8, count=width * height, offset=pos).reshape(height, width)


def read_raster(path) -> np.ndarray:
    """The image as stored: uint8 (H, W).  PGM (P5, maxval 255) or 8-bit grayscale PNG (converted
    to mode "L" like load_image)."""
    path = Path(path)
    if path.suffix.lower() == ".png":
        from PIL import Image as PILImage
        with PILImage.open(path) as im:
            return np.asarray(im if im.mode == "L" else im.convert("L"), dtype=np.uint8)
    return _parse_pgm(path, path.read_bytes())


def quantize(img) -> np.ndarray:
    """8-bit raster of a float image: floor(clip(x, 0, 255) + 0.5) (image.py:96-99)."""
    if isinstance(img, np.ndarray) and img.dtype == np.uint8:
        return img
    return np.floor(np.clip(as_image(img), 0.0, 255.0) + 0.5).astype(np.uint8)


def write_raster(path, raster: np.ndarray) -> None:
    """Write a uint8 raster as binary PGM, or PNG when the suffix is .png."""
    raster = np.ascontiguousarray(raster, dtype=np.uint8)
    path = Path(path)
    if path.suffix.lower() == ".png":
        from PIL import Image as PILImage
        PILImage.fromarray(raster, mode="L").save(path)
        return
    h, w = raster.shape
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n255\n" % (w, h))
        fh.write(raster.tobytes())


def load_pgm(path) -> np.ndarray:
    """Binary 8-bit PGM as a float64 image (image.py:73-93)."""
    return _parse_pgm(path, Path(path).read_bytes()).astype(np.float64)


def save_pgm(path, img) -> None:
    """Binary 8-bit PGM, clamped to [0, 255] and rounded half up (image.py:96-102)."""
    raster = quantize(img)
    h, w = raster.shape
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n255\n" % (w, h))
        fh.write(np.ascontiguousarray(raster).tobytes())


def load_image(path) -> np.ndarray:
    """PGM or 8-bit grayscale PNG as a float64 image (image.py:105-114)."""
    return read_raster(path).astype(np.float64)


def save_image(path, img) -> None:
    """PGM or PNG by suffix, with save_pgm's quantisation (image.py:117-129)."""
    write_raster(path, quantize(img))
