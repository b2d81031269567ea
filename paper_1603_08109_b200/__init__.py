"""B200-native GPA bilateral filter (arXiv 1603.08109) — drop-in for `fastbilateral`'s filter path.

The public names mirror `/root/reference/pkg/src/fastbilateral/__init__.py:35-48`
for the hot path (§8 of SURVEY.md): the filter (`gpa_filter`,
`gpa_filter_auto`), the spatial filters it applies (`apply_spatial`,
`box_filter`, `gaussian_filter`, `convolve_direct`), kernels, range handling,
order selection and the error types; and the tools around it (§8(f)): the
exact filter, error metrology (`analysis`), PGM/PNG I/O and the CLI (`cli`).  Filtering runs in hand-written sm_100a CUDA kernels
(`csrc/`, loaded from the in-tree `libfbgpu.so` through `_native`); there is
no CPU fallback.
"""

import os as _os

# FASTBILATERAL_THREADS caps the host's numeric thread pools (numpy/BLAS in the host-side helpers)
# before numpy is first imported, as the reference package does (fastbilateral/__init__.py:10-16).
_threads = _os.environ.get("FASTBILATERAL_THREADS")
if _threads:
    for _name in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        _os.environ.setdefault(_name, _threads)

from .analysis import (ErrorReport, accuracy_bound, error_report, kernel_error_sup, linf_error, mse_db,
                       psi_eval)
from .conv import apply_spatial, box_filter, convolve_direct, gaussian_filter
from .engine import gpa_filter, gpa_filter_auto, gpa_filter_batch
from .errors import (BoundInapplicableError, NativeError, NumericRangeError, ParameterError,
                     RangeViolationError)
from .image import (RANGE_8BIT, RangeSpec, as_image, center, load_image, load_pgm, quantize, read_raster,
                    save_image, save_pgm, uncenter, validate_range, write_raster)
from .kernels import SpatialKernel, gauss_poly, make_spatial_kernel, range_kernel
from .reference import bilateral_exact
from .order import (OrderEstimate, chebyshev_order, chernoff_order_exhaustive, epsilon_from_delta,
                    estimate_order, lambert_w0_series, log_chernoff, order_approx, poisson_tail, yang_order)

__version__ = "1.0.0"

__all__ = [
    "ErrorReport", "OrderEstimate", "RangeSpec", "SpatialKernel", "RANGE_8BIT", "__version__",
    "accuracy_bound", "apply_spatial", "as_image", "bilateral_exact", "box_filter", "center",
    "chebyshev_order", "chernoff_order_exhaustive", "convolve_direct", "epsilon_from_delta", "error_report",
    "estimate_order", "gauss_poly", "gaussian_filter", "gpa_filter", "gpa_filter_auto", "gpa_filter_batch",
    "kernel_error_sup", "lambert_w0_series", "linf_error", "load_image", "load_pgm", "log_chernoff",
    "make_spatial_kernel", "mse_db", "order_approx", "poisson_tail", "psi_eval", "quantize", "range_kernel",
    "read_raster", "save_image", "save_pgm", "uncenter", "validate_range", "write_raster", "yang_order",
    "BoundInapplicableError", "NativeError", "NumericRangeError", "ParameterError",
    "RangeViolationError",
]
