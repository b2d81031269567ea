"""Single-channel spatial filters on the GPU (box / separable Gaussian, replicate boundary).

Mirrors `/root/reference/pkg/src/fastbilateral/conv.py:43-80` (`box_filter`,
`gaussian_filter`, `apply_spatial`): the same kernels the GPA path applies to
each channel, exposed for one image.  They run the same two CUDA kernels in
"plain" mode (channel = the image itself, no Horner epilogue).  Default
precision is fp64 so results agree with the reference's fp64 numpy filters to
~1e-12; `precision="f32"` is available for large images.
`convolve_direct` (`conv.py:83-96`), the literal O(W^2) double sum with the 2-D weight table that
the reference uses as its convolution oracle, runs as its own device kernel
(`fb_convolve_direct`), accumulated in the reference's order without FMA contraction.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .engine import _alloc_out, _coerce, _shape_check, _window_error, _PREC
from .errors import ParameterError
from .kernels import SpatialKernel, make_spatial_kernel


def _run(img, kernel: SpatialKernel, precision: str, device, check_window: bool):
    a, is_dev = _coerce(img)
    shape = _shape_check(a)
    dev = _native.device_of(a, device)
    if check_window:
        err = _window_error(kernel, shape) if kernel.kind == "box" else _gauss_window_error(kernel, shape)
        if err is not None:
            _native.validate(a, -np.inf, np.inf, dev)
            raise err
    if precision not in _PREC:
        raise ParameterError(f"precision must be 'f32' or 'f64', got {precision!r}")
    out = _alloc_out(a, is_dev, shape, np.float64)
    _native.spatial(a, out, kernel, _PREC[precision], dev)
    return out


def _gauss_window_error(kernel, shape):
    limit = min((d for d in shape if d > 1), default=1)
    if kernel.half_width >= limit:
        return ParameterError(
            f"window half-width {kernel.half_width} too large for {shape[0]}x{shape[1]} image")
    return None


def box_filter(img, W: int, *, precision: str = "f64", device: int | None = None):
    """Normalised (2W+1)^2 box filter, replicate boundary (conv.py:43-54)."""
    try:
        ok = int(W) == W and W >= 1
    except (TypeError, ValueError, OverflowError):
        ok = False
    if not ok:
        raise ParameterError(f"W must be an integer >= 1, got {W}")
    return _run(img, make_spatial_kernel("box", half_width=int(W)), precision, device, True)


def gaussian_filter(img, sigma_s: float, *, precision: str = "f64", device: int | None = None):
    """Separable truncated Gaussian on [-W, W], W = ceil(3 sigma_s) (conv.py:67-72)."""
    return _run(img, make_spatial_kernel("gaussian", sigma_s=sigma_s), precision, device, True)


def apply_spatial(img, kernel: SpatialKernel, *, precision: str = "f64", device: int | None = None):
    """Filter with a constructed kernel (conv.py:75-80): box checks its window, Gaussian does not."""
    return _run(img, kernel, precision, device, kernel.kind == "box")


def convolve_direct(img, kernel: SpatialKernel, *, device: int | None = None):
    """Literal double-sum convolution out(i) = sum_j w(j) img(i - j), 2-D table, replicate boundary
    (conv.py:83-96); fp64, float64 result.  The window check applies to every kernel kind."""
    a, is_dev = _coerce(img)
    shape = _shape_check(a)
    dev = _native.device_of(a, device)
    err = _gauss_window_error(kernel, shape)
    if err is not None:
        _native.validate(a, -np.inf, np.inf, dev)
        raise err
    out = _alloc_out(a, is_dev, shape, np.float64)
    _native.convolve_direct(a, out, kernel.weights, kernel.half_width, dev)
    return out
