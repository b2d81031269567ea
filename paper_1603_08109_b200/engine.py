"""The drop-in filter API: `gpa_filter` / `gpa_filter_auto` on B200 kernels.

Same names, arguments, defaults, return types, exceptions and `stats` keys as
the reference (`/root/reference/pkg/src/fastbilateral/engine.py:27-98`); the
work runs in `libfbgpu.so` (two kernels per row band):

  gpa_filter(img, spatial, sigma_r, order, range_spec=None, *,
             allow_small_sigma=False, stats=None)            -> float64 ndarray
  gpa_filter_auto(img, spatial, sigma_r, delta, range_spec=None, *,
                  allow_small_sigma=False, stats=None)       -> (ndarray, OrderEstimate)

Extensions (keyword-only, defaulted so reference call sites are unchanged):

* `precision`: "auto" (default), "f32" or "f64".  "auto" runs fp64 for
  images of at most 65,536 pixels (launch-latency bound, where fp64 costs
  nothing and the reference suite's 1e-6 / 1e-9 tolerances apply) and for
  sigma_r < 16 (where fp32 channels could underflow/overflow); fp32 otherwise
  (max |delta| vs the fp64 reference <= 1e-3 gray levels, tests/test_gpu_parity.py).
* `out`: optional preallocated float32/float64 output (numpy for numpy input, e.g.
  pinned memory; CUDA tensor for tensor input).
* `device`: CUDA device index for numpy inputs.  A CUDA torch tensor input is
  filtered where it lives and the result is returned as a CUDA float64 tensor
  (or `out_dtype`), without host copies.

Check order follows the reference: shape, finiteness and range
(`image.py:35-54`), then sigma_r (`engine.py:40-46`), order (`engine.py:47-49`),
and the box window (`conv.py:19-27`, raised by the first spatial filtering).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import ParameterError
from .image import RangeSpec
from .kernels import SpatialKernel
from .order import OrderEstimate, epsilon_from_delta, estimate_order

#: |Q| below this passes the input pixel through (engine.py:20).
Q_FLOOR = 1e-30
#: sigma_r floor without `allow_small_sigma` (engine.py:24).
SIGMA_R_FLOOR = 10.0
#: "auto" precision: fp64 at or below this many pixels, or below this sigma_r.
AUTO_F64_MAX_PIXELS = 65536
AUTO_F64_SIGMA_R = 16.0

_PREC = {"f32": _native.FB_PREC_F32, "f64": _native.FB_PREC_F64}


def _coerce(img):
    """(array, is_device): numpy (uint8/float32/float64, unit-stride rows) or a CUDA torch tensor."""
    if _native.is_cuda_tensor(img):
        t = img
        if str(t.dtype) not in ("torch.uint8", "torch.float32", "torch.float64"):
            t = t.double()
        if t.dim() == 2 and t.numel() and t.stride(1) != 1:
            t = t.contiguous()
        return t, True
    if type(img).__module__.startswith("torch"):
        img = img.detach().cpu().numpy()
    a = np.asarray(img)
    if a.dtype not in (np.uint8, np.float32, np.float64):
        a = np.asarray(a, dtype=np.float64)
    if a.ndim == 2 and a.size and (a.strides[1] != a.itemsize or a.strides[0] < a.shape[1] * a.itemsize):
        a = np.ascontiguousarray(a)
    return a, False


def _shape_check(a) -> tuple[int, int]:
    shape = tuple(a.shape)
    n = 1
    for d in shape:
        n *= d
    if len(shape) != 2 or n == 0:
        raise ParameterError(f"image must be a non-empty 2-D array, got shape {shape}")
    return shape


def _window_error(kernel: SpatialKernel, shape) -> ParameterError | None:
    if kernel.kind != "box":
        return None
    limit = min((d for d in shape if d > 1), default=1)
    if kernel.half_width >= limit:
        return ParameterError(
            f"window half-width {kernel.half_width} too large for {shape[0]}x{shape[1]} image")
    return None


def resolve_precision(precision: str, shape, sigma_r: float) -> int:
    if precision == "auto":
        small = shape[0] * shape[1] <= AUTO_F64_MAX_PIXELS
        return _native.FB_PREC_F64 if (small or sigma_r < AUTO_F64_SIGMA_R) else _native.FB_PREC_F32
    try:
        return _PREC[precision]
    except KeyError:
        raise ParameterError(f"precision must be 'auto', 'f32' or 'f64', got {precision!r}") from None


def _alloc_out(a, is_dev: bool, shape, out_dtype):
    if is_dev:
        import torch
        return torch.empty(shape, dtype=getattr(torch, np.dtype(out_dtype).name), device=a.device)
    return np.empty(shape, dtype=out_dtype)


def gpa_filter(img, spatial: SpatialKernel, sigma_r: float, order: int,
               range_spec: RangeSpec | None = None, *, allow_small_sigma: bool = False,
               stats: dict | None = None, precision: str = "auto", device: int | None = None,
               out_dtype=np.float64, out=None):
    """Approximate bilateral filter of order N (Algorithm 2) on the GPU; returns float64 (H, W)."""
    a, is_dev = _coerce(img)
    shape = _shape_check(a)
    if range_spec is None:
        range_spec = RangeSpec(half_range=128.0, center=128.0)
    dev = _native.device_of(a, device)

    param_error = None
    if not sigma_r > 0:
        param_error = ParameterError(f"sigma_r must be positive, got {sigma_r}")
    elif sigma_r < SIGMA_R_FLOOR and not allow_small_sigma:
        param_error = ParameterError(
            f"sigma_r = {sigma_r} below {SIGMA_R_FLOOR}; intermediate images may "
            "overflow (pass allow_small_sigma=True to override)")
    else:
        try:
            ok = int(order) == order and order >= 1
        except (TypeError, ValueError, OverflowError):
            ok = False
        if not ok:
            param_error = ParameterError(f"order must be an integer >= 1, got {order}")
        else:
            param_error = _window_error(spatial, shape)
    if param_error is not None:
        # Input errors take precedence (the reference validates the image first).
        _native.validate(a, range_spec.lo, range_spec.hi, dev)
        raise param_error

    prec = resolve_precision(precision, shape, sigma_r)
    if out is None:
        out = _alloc_out(a, is_dev, shape, out_dtype)
    elif tuple(out.shape) != shape or _native.is_cuda_tensor(out) != is_dev:
        raise ParameterError("out must match the image shape and live where the image lives")
    st = _native.gpa(a, out, spatial, float(sigma_r), int(order), range_spec.center,
                     range_spec.half_range, prec, dev)
    if stats is not None:
        stats["spatial_filter_calls"] = int(order) + 1
        stats["order"] = int(order)
        stats["degenerate_pixels"] = st["degenerate_pixels"]
        stats["precision"] = "f64" if st["precision"] == _native.FB_PREC_F64 else "f32"
        stats["device_ms"] = st["device_ms"]
        stats["kernel_ms"] = st["kernel_ms"]
        stats["k1_ms"] = st["k1_ms"]
        stats["k2_ms"] = st["k2_ms"]
        stats["launches"] = st["launches"]
        stats["bands"] = st["bands"]
        stats["h2d_bytes"] = st["h2d_bytes"]
        stats["d2h_bytes"] = st["d2h_bytes"]
    return out


def gpa_filter_batch(images, spatial: SpatialKernel, sigma_r: float, order: int,
                     range_spec: RangeSpec | None = None, *, allow_small_sigma: bool = False,
                     stats: dict | None = None, precision: str = "auto", device: int | None = None,
                     out_dtype=np.float64, outs=None) -> list:
    """`gpa_filter` over a batch of equally wide images in one call (by-image partitioning, config c3).

    Host-resident images are pipelined (copy-in of image i+1 and copy-out of image i-1 overlap
    the kernels of image i).  Returns the list of outputs; errors name the offending image.
    """
    arrs = [_coerce(im) for im in images]
    if not arrs:
        return []
    is_dev = arrs[0][1]
    if any(d != is_dev for _, d in arrs):
        raise ParameterError("a batch must be all host arrays or all CUDA tensors")
    arrs = [a for a, _ in arrs]
    shapes = [_shape_check(a) for a in arrs]
    if len({s[1] for s in shapes}) != 1:
        raise ParameterError("images of a batch must share their width")
    if range_spec is None:
        range_spec = RangeSpec(half_range=128.0, center=128.0)
    if not (sigma_r > 0) or (sigma_r < SIGMA_R_FLOOR and not allow_small_sigma) or \
            not (isinstance(order, (int, np.integer)) or float(order).is_integer()) or order < 1 or \
            any(_window_error(spatial, s) for s in shapes):
        # single-image path raises exactly the reference's errors in the reference's order
        for a in arrs:
            gpa_filter(a, spatial, sigma_r, order, range_spec, allow_small_sigma=allow_small_sigma,
                       precision=precision, device=device)
    dev = _native.device_of(arrs[0], device)
    prec = resolve_precision(precision, min(shapes, key=lambda s: s[0] * s[1]), sigma_r)
    if outs is None:
        outs = [_alloc_out(a, is_dev, s, out_dtype) for a, s in zip(arrs, shapes)]
    st = _native.gpa_batch(arrs, outs, spatial, float(sigma_r), int(order), range_spec.center,
                           range_spec.half_range, prec, dev)
    if stats is not None:
        stats.update({k: st[k] for k in ("degenerate_pixels", "device_ms", "kernel_ms", "k1_ms", "k2_ms",
                                         "launches", "bands", "h2d_bytes", "d2h_bytes")})
        stats["spatial_filter_calls"] = int(order) + 1
        stats["order"] = int(order)
        stats["precision"] = "f64" if st["precision"] == _native.FB_PREC_F64 else "f32"
    return outs


def gpa_filter_auto(img, spatial: SpatialKernel, sigma_r: float, delta: float,
                    range_spec: RangeSpec | None = None, *, allow_small_sigma: bool = False,
                    stats: dict | None = None, **kw) -> tuple[np.ndarray, OrderEstimate]:
    """Filter to within +-delta of the exact bilateral filter: delta -> eps -> N, then `gpa_filter`."""
    if range_spec is None:
        range_spec = RangeSpec(half_range=128.0, center=128.0)
    eps = epsilon_from_delta(delta, spatial.w0, range_spec.half_range)
    est = estimate_order(sigma_r, eps, range_spec.half_range)
    out = gpa_filter(img, spatial, sigma_r, est.N0, range_spec,
                     allow_small_sigma=allow_small_sigma, stats=stats, **kw)
    return out, est
