"""Error metrology: image differences, the kernel-error grid search and the accuracy bound.

Restates `/root/reference/pkg/src/fastbilateral/analysis.py:1-118`.  The
data-parallel parts run on the GPU through the C ABI:

* `linf_error`, `mse_db`, `error_report` (`analysis.py:28-52`): one fp64 reduction kernel over
  both images (`fb_error_stats`), with `as_image`'s finiteness check fused in.  Inputs are numpy
  arrays (copied in) or CUDA tensors (read where they are), so the full-size error reports of the
  `compare` command never leave the device.  linf is exact; the mean of squares is a blocked fp64
  sum (numpy sums pairwise), equal to ~1e-15 relative.
* `kernel_error_sup` (`analysis.py:70-103`): one device thread per grid point (t, tau) evaluating
  the tail series (`fb_kernel_error_sup`).
* `psi_eval` and `accuracy_bound` (`analysis.py:55-67`, `:106-118`) are scalar formulas (host).

Argument checks, their order and the exception types/messages follow the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import BoundInapplicableError, ParameterError
from .order import poisson_tail


@dataclass
class ErrorReport:
    """Difference metrics between two images plus optional bound values (analysis.py:15-25)."""

    linf: float
    linf_db: float  # 20 log10(linf); -inf when the images agree
    mse_db: float   # 10 log10(mean squared difference); -inf on equality
    kernel_error_sup: float | None = None
    kernel_bound: float | None = None
    accuracy_bound: float | None = None
    runtime_ms: dict = field(default_factory=dict)


def _as_2d(x):
    """as_image's shape rule (image.py:37-39) without the host float64 copy."""
    if _native.is_cuda_tensor(x):
        if x.dim() != 2 or x.numel() == 0:
            raise ParameterError(f"image must be a non-empty 2-D array, got shape {tuple(x.shape)}")
        if str(x.dtype) not in ("torch.uint8", "torch.float32", "torch.float64"):
            x = x.double()
        return x.contiguous() if x.stride(1) != 1 else x
    if type(x).__module__.startswith("torch"):
        x = x.detach().cpu().numpy()
    a = np.asarray(x)
    if a.dtype not in (np.uint8, np.float32, np.float64):
        a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.size == 0:
        raise ParameterError(f"image must be a non-empty 2-D array, got shape {a.shape}")
    if a.strides[1] != a.itemsize or a.strides[0] < a.shape[1] * a.itemsize:
        a = np.ascontiguousarray(a)
    return a


def _diff_stats(a, b) -> tuple[float, float, int]:
    """(max |a - b|, sum (a - b)^2, pixel count) on the device; reference check order:
    a's shape and finiteness, b's shape and finiteness, then equal shapes (analysis.py:28-31)."""
    a = _as_2d(a)
    try:
        b = _as_2d(b)
    except ParameterError:
        _native.validate(a, -np.inf, np.inf, _native.device_of(a, None))
        raise
    dev = _native.device_of(a, None)
    if tuple(a.shape) != tuple(b.shape):
        _native.validate(a, -np.inf, np.inf, dev)
        _native.validate(b, -np.inf, np.inf, _native.device_of(b, None))
        raise ParameterError(f"image dimensions differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    if _native.is_cuda_tensor(a) != _native.is_cuda_tensor(b):
        # one operand on the device, one on the host: bring the host one over
        import torch
        if _native.is_cuda_tensor(a):
            b = torch.from_numpy(np.ascontiguousarray(b)).to(a.device)
        else:
            a = torch.from_numpy(np.ascontiguousarray(a)).to(b.device)
            dev = _native.device_of(a, None)
    linf, ss = _native.error_stats(a, b, dev)
    return linf, ss, int(a.shape[0]) * int(a.shape[1])


def linf_error(a, b) -> float:
    """Maximum absolute per-pixel difference (analysis.py:33-37)."""
    return _diff_stats(a, b)[0]


def _mse_db_from(ss: float, n: int) -> float:
    m = ss / n
    return -math.inf if m == 0.0 else 10.0 * math.log10(m)


def mse_db(a, b) -> float:
    """Mean squared difference in decibels (10 log10); -inf on exact equality (analysis.py:40-45)."""
    _, ss, n = _diff_stats(a, b)
    return _mse_db_from(ss, n)


def error_report(a, b) -> ErrorReport:
    """linf, 20 log10 linf and mse_db of two images from one device pass (analysis.py:48-52)."""
    linf, ss, n = _diff_stats(a, b)
    linf_db = -math.inf if linf == 0.0 else 20.0 * math.log10(linf)
    return ErrorReport(linf=linf, linf_db=linf_db, mse_db=_mse_db_from(ss, n))


def psi_eval(s: float, N: int, sigma_r: float) -> float:
    """Poisson(s / sigma_r^2) tail beyond N, the tail weight at product value s >= 0 (analysis.py:55-67)."""
    if not (s >= 0):
        raise ParameterError(f"s must be nonnegative, got {s}")
    if not (sigma_r > 0):
        raise ParameterError(f"sigma_r must be positive, got {sigma_r}")
    if s == 0.0:
        return 0.0 if N >= 1 else 1.0
    return poisson_tail(N, s / sigma_r**2)


def kernel_error_sup(N: int, sigma_r: float, T: float, *, device: int = 0) -> float:
    """Worst-case kernel error over the integer grid t, tau in {-T..T} (analysis.py:70-103), on the GPU."""
    if N < 1:
        raise ParameterError(f"N must be >= 1, got {N}")
    if not (sigma_r > 0 and T > 0):
        raise ParameterError("sigma_r and T must be positive")
    return _native.kernel_error_sup(int(N), float(sigma_r), float(T), device)


def accuracy_bound(kernel_err: float, w0: float, T: float) -> float:
    """Worst-case filtering error implied by a kernel error: 2 T e / (w0 - e) (analysis.py:106-118)."""
    if not (kernel_err >= 0):
        raise ParameterError(f"kernel_err must be nonnegative, got {kernel_err}")
    if not (0.0 < w0 <= 1.0):
        raise ParameterError(f"w0 must lie in (0, 1], got {w0}")
    if not (T > 0):
        raise ParameterError(f"T must be positive, got {T}")
    if kernel_err >= w0:
        raise BoundInapplicableError(f"kernel error {kernel_err} >= center weight {w0}; bound is vacuous")
    return 2.0 * T * kernel_err / (w0 - kernel_err)
