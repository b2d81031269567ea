"""Tail probabilities and the order estimates the CLI's `order` command reports beside Algorithm 1.

Restates `/root/reference/pkg/src/fastbilateral/order.py:37-68` and `:156-184`:

* `poisson_tail(N, lam)`: P[X >= N] for X ~ Poisson(lam), as one minus the head of the series
  (terms by the ratio recursion t_n = t_{n-1} lam / n, summed in order), clamped to [0, 1];
* `chebyshev_order(lam, eps)`: ceil(lam + sqrt(lam / eps));
* `order_approx(sigma_r, delta, w0, T)`: the closed form 1.72 lam + ln(2T / (w0 delta));
* `yang_order(sigma_r, delta)`: 1.14e5 / (sqrt(delta) sigma_r^2), a comparator only.

The last two round to nearest with halves up.  Scalar host code; the floating-point operations
and their order are the reference's, so the values agree bit for bit
(`tests/test_tools_host.py` against reference-generated fixtures).
"""

from __future__ import annotations

import math

from .errors import ParameterError
from .order import OrderEstimate, _require_eps, _require_lambda


def poisson_tail(N: int, lam: float) -> float:
    if not lam > 0:
        raise ParameterError(f"lambda must be positive, got {lam}")
    if N < 0:
        raise ParameterError(f"N must be nonnegative, got {N}")
    if N == 0:
        return 1.0
    head = term = math.exp(-lam)
    n = 1
    while n < N:
        term = term * (lam / n)
        head = head + term
        n += 1
    tail = 1.0 - head
    return 1.0 if tail > 1.0 else (0.0 if tail < 0.0 else tail)


def chebyshev_order(lam: float, epsilon: float) -> OrderEstimate:
    _require_eps(epsilon)
    _require_lambda(lam)
    n0 = math.ceil(lam + math.sqrt(lam / epsilon))
    return OrderEstimate(N0=n0, method="chebyshev", epsilon=epsilon, lam=lam)


def _half_up(v: float) -> int:
    return math.floor(v + 0.5)


def order_approx(sigma_r: float, delta: float, w0: float, T: float) -> OrderEstimate:
    if sigma_r <= 0 or delta <= 0 or T <= 0 or math.isnan(sigma_r + delta + T):
        raise ParameterError("sigma_r, delta and T must be positive")
    if not 0.0 < w0 <= 1.0:
        raise ParameterError(f"w0 must lie in (0, 1], got {w0}")
    lam = (T / sigma_r) ** 2
    estimate = 1.72 * lam + math.log(2.0 * T / (w0 * delta))
    return OrderEstimate(N0=_half_up(estimate), method="approx_formula", lam=lam)


def yang_order(sigma_r: float, delta: float) -> OrderEstimate:
    if sigma_r <= 0 or delta <= 0 or math.isnan(sigma_r + delta):
        raise ParameterError("sigma_r and delta must be positive")
    return OrderEstimate(N0=_half_up(1.14e5 / (math.sqrt(delta) * sigma_r**2)), method="yang_formula")
