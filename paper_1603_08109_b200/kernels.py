"""Spatial kernels consumed by the filter.

Host-side construction of the normalised box / truncated-Gaussian spatial
kernel, restating `make_spatial_kernel` and `SpatialKernel`
(`/root/reference/pkg/src/fastbilateral/kernels.py:13-31`, `:61-86`):

* box, half-width W: uniform weight 1/(2W+1)^2 on [-W, W]^2, 1-D factor 1/(2W+1);
* gaussian, sigma_s: W = ceil(3 sigma_s), 1-D taps exp(-k^2 / 2 sigma_s^2)
  normalised to sum 1, 2-D weights = normalised outer product.

The GPU kernels only consume `half_width` and `weights_1d` (the separable
factor); the 2-D table is kept because `w0` (the centre weight) drives the
order selection of `gpa_filter_auto`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import ParameterError


@dataclass(frozen=True)
class SpatialKernel:
    """Normalised nonnegative weights on the square window [-W, W]^2.

    `weights[W, W]` is the origin; `weights_1d` is the normalised separable
    factor with `outer(weights_1d, weights_1d) == weights` (to rounding).
    """

    kind: str
    half_width: int
    weights: np.ndarray = field(repr=False)
    weights_1d: np.ndarray = field(repr=False)
    sigma_s: float | None = None

    @property
    def w0(self) -> float:
        """Centre weight w(0), the quantity the accuracy bound depends on."""
        c = self.half_width
        return float(self.weights[c, c])


def _box(half_width) -> SpatialKernel:
    if half_width is None or half_width < 1 or int(half_width) != half_width:
        raise ParameterError(f"box kernel needs integer half_width >= 1, got {half_width}")
    W = int(half_width)
    side = 2 * W + 1
    taps = np.full(side, 1.0 / side)
    table = np.full((side, side), 1.0 / (side * side))
    return SpatialKernel("box", W, table, taps)


def _gaussian(sigma_s) -> SpatialKernel:
    if sigma_s is None or not sigma_s > 0:
        raise ParameterError(f"gaussian kernel needs sigma_s > 0, got {sigma_s}")
    W = int(math.ceil(3.0 * sigma_s))
    k = np.arange(-W, W + 1, dtype=np.float64)
    g = np.exp(-(k * k) / (2.0 * sigma_s * sigma_s))
    table = g[:, None] * g[None, :]
    table = table / table.sum()
    return SpatialKernel("gaussian", W, table, g / g.sum(), float(sigma_s))


def make_spatial_kernel(kind: str, *, sigma_s: float | None = None,
                        half_width: int | None = None) -> SpatialKernel:
    """Build a box (`half_width=W`) or truncated Gaussian (`sigma_s=...`) kernel."""
    if kind == "box":
        return _box(half_width)
    if kind == "gaussian":
        return _gaussian(sigma_s)
    raise ParameterError(f"unknown spatial kernel kind {kind!r}")


def range_kernel(t, sigma_r: float):
    """Gaussian range kernel exp(-t^2 / (2 sigma_r^2)), elementwise (kernels.py:33-37)."""
    if not sigma_r > 0:
        raise ParameterError(f"sigma_r must be positive, got {sigma_r}")
    t = np.asarray(t, dtype=np.float64)
    return np.exp(-np.square(t) / (2.0 * sigma_r**2))


def gauss_poly(t: float, tau: float, order: int, sigma_r: float) -> float:
    """Order-N approximant of the translated range kernel (kernels.py:40-58):
    exp(-(t^2 + tau^2) / 2 sigma_r^2) times the first `order` Taylor terms of exp(t tau / sigma_r^2),
    summed by the term recursion (no factorials)."""
    if not sigma_r > 0:
        raise ParameterError(f"sigma_r must be positive, got {sigma_r}")
    if order < 1:
        raise ParameterError(f"order must be >= 1, got {order}")
    x = (t * tau) / sigma_r**2
    term = acc = 1.0
    for n in range(1, order):
        term *= x / n
        acc += term
    return math.exp(-(t * t + tau * tau) / (2.0 * sigma_r**2)) * acc
