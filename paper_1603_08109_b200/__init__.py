"""B200-native GPA bilateral filter (arXiv 1603.08109) — drop-in for `fastbilateral`'s filter path.

The public names mirror `/root/reference/pkg/src/fastbilateral/__init__.py:35-48`
for the hot path (§8 of SURVEY.md): the filter (`gpa_filter`,
`gpa_filter_auto`), the spatial filters it applies (`apply_spatial`,
`box_filter`, `gaussian_filter`), kernels, range handling, order selection and
the error types.  Filtering runs in hand-written sm_100a CUDA kernels
(`csrc/`, loaded from the in-tree `libfbgpu.so` through `_native`); there is
no CPU fallback.
"""

from .conv import apply_spatial, box_filter, gaussian_filter
from .engine import gpa_filter, gpa_filter_auto, gpa_filter_batch
from .errors import (BoundInapplicableError, NativeError, NumericRangeError, ParameterError,
                     RangeViolationError)
from .image import RANGE_8BIT, RangeSpec, as_image, center, uncenter, validate_range
from .kernels import SpatialKernel, make_spatial_kernel
from .reference import bilateral_exact
from .order import (OrderEstimate, chernoff_order_exhaustive, epsilon_from_delta, estimate_order,
                    lambert_w0_series, log_chernoff)

__version__ = "1.0.0"

__all__ = [
    "OrderEstimate", "RangeSpec", "SpatialKernel", "RANGE_8BIT", "__version__",
    "apply_spatial", "as_image", "bilateral_exact", "box_filter", "center", "chernoff_order_exhaustive",
    "epsilon_from_delta", "estimate_order", "gaussian_filter", "gpa_filter", "gpa_filter_auto",
    "gpa_filter_batch",
    "lambert_w0_series", "log_chernoff", "make_spatial_kernel", "uncenter", "validate_range",
    "BoundInapplicableError", "NativeError", "NumericRangeError", "ParameterError",
    "RangeViolationError",
]
