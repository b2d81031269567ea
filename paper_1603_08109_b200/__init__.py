"""B200-native GPA bilateral filter (arXiv 1603.08109): a drop-in for `fastbilateral`.

Every public name of the reference package (`/root/reference/pkg/src/fastbilateral/__init__.py`)
is exported here, grouped below by the module that implements it:

* the filter path: `gpa_filter`, `gpa_filter_auto` (+ `gpa_filter_batch`), the
  spatial filters it applies, the kernels, range handling, order selection and the error types;
* the tools around it (§8(f)): the exact filter, error metrology, PGM/PNG I/O and the CLI
  (`python -m paper_1603_08109_b200`).

Filtering runs in hand-written sm_100a CUDA kernels (`csrc/`, the in-tree `libfbgpu.so` reached
through `_native`); there is no CPU fallback.
"""

import importlib as _importlib
import os as _os

# FASTBILATERAL_THREADS caps the host's numeric thread pools (numpy/BLAS in the host-side helpers)
# before numpy is first imported, as the reference package does (fastbilateral/__init__.py:10-16).
if _os.environ.get("FASTBILATERAL_THREADS"):
    for _pool in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        _os.environ.setdefault(_pool, _os.environ["FASTBILATERAL_THREADS"])

__version__ = "1.0.0"

# implementing module -> the names it contributes to the package namespace
_PUBLIC = {
    "engine": "gpa_filter gpa_filter_auto gpa_filter_batch",
    "conv": "apply_spatial box_filter convolve_direct gaussian_filter",
    "kernels": "SpatialKernel gauss_poly make_spatial_kernel range_kernel",
    "image": "RANGE_8BIT RangeSpec as_image center load_image load_pgm quantize read_raster save_image "
             "save_pgm uncenter validate_range write_raster",
    "order": "OrderEstimate chebyshev_order chernoff_order_exhaustive epsilon_from_delta estimate_order "
             "lambert_w0_series log_chernoff order_approx poisson_tail yang_order",
    "analysis": "ErrorReport accuracy_bound error_report kernel_error_sup linf_error mse_db psi_eval",
    "reference": "bilateral_exact",
    "errors": "BoundInapplicableError NativeError NumericRangeError ParameterError RangeViolationError",
}

for _mod, _names in _PUBLIC.items():
    _m = _importlib.import_module(f".{_mod}", __name__)
    for _n in _names.split():
        globals()[_n] = getattr(_m, _n)

__all__ = sorted(n for names in _PUBLIC.values() for n in names.split()) + ["__version__"]

del _importlib, _os, _mod, _names, _m, _n
