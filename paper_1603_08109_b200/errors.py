"""Exception types of the drop-in API.

Mirrors the reference's error convention (`/root/reference/pkg/src/fastbilateral/errors.py:4-17`):
the class names, base classes and meanings are the same so that callers that
catch `ParameterError` (a `ValueError`) or `NumericRangeError` (an
`ArithmeticError`) keep working when they switch to this package.  The native
C-ABI reports the same conditions as integer status codes
(`include/fbgpu.h`, `FB_ERR_*`), translated back to these classes in
`_native.py`.
"""


class ParameterError(ValueError):
    """Invalid parameter or input shape (nonpositive sigma, bad order, window too large, ...)."""


class RangeViolationError(ValueError):
    """An input sample lies outside the declared intensity range."""


class BoundInapplicableError(ValueError):
    """The filtering-accuracy bound is vacuous (kernel error >= centre weight)."""


class NumericRangeError(ArithmeticError):
    """The filter produced non-finite output (intermediates left the representable range)."""


class NativeError(RuntimeError):
    """The CUDA library failed (missing extension, CUDA runtime error, out of device memory)."""
