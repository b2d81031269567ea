"""Exact O(W^2) bilateral filter on the GPU (fp64): the approximation-error oracle.

Mirrors `bilateral_exact` (`/root/reference/pkg/src/fastbilateral/reference.py:17-45`):
out(i) = sum_j w(j) g(f(i-j) - f(i)) f(i-j) / sum_j w(j) g(f(i-j) - f(i)), replicate
boundary, fp64.  Same argument checks and exceptions.  It is a measurement tool (the GPA error
reports of DESIGN.md §2 at full image size), not part of the filter path.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .engine import _alloc_out, _coerce, _shape_check
from .errors import ParameterError
from .kernels import SpatialKernel


def bilateral_exact(img, spatial: SpatialKernel, sigma_r: float, *, device: int | None = None):
    a, is_dev = _coerce(img)
    shape = _shape_check(a)
    dev = _native.device_of(a, device)
    W = spatial.half_width
    err = None
    if not sigma_r > 0:
        err = ParameterError(f"sigma_r must be positive, got {sigma_r}")
    elif W >= min(shape):
        err = ParameterError(f"window half-width {W} too large for {shape[0]}x{shape[1]} image")
    # as_image (finite samples only) runs first in the reference (reference.py:24), so a bad image
    # is reported before a bad parameter
    _native.validate(a, -np.inf, np.inf, dev)
    if err is not None:
        raise err
    out = _alloc_out(a, is_dev, shape, np.float64)
    _native.bilateral_exact(a, out, spatial, float(sigma_r), dev)
    return out
