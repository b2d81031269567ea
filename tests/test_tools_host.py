"""Host-side scalar tools vs the reference's values: order comparators, Poisson tail, psi,
accuracy bound, range kernel and its polynomial approximant (CPU)."""

import math

import numpy as np
import pytest

from paper_1603_08109_b200 import (BoundInapplicableError, ParameterError, accuracy_bound, chebyshev_order,
                                   epsilon_from_delta, gauss_poly, order_approx, poisson_tail, psi_eval,
                                   range_kernel, yang_order)


def test_poisson_tail(tools_scalars):
    for n, lam, v in tools_scalars["poisson_tail"]:
        assert poisson_tail(n, lam) == v, (n, lam)


def test_psi_eval(tools_scalars):
    for s, n, sr, v in tools_scalars["psi_eval"]:
        assert psi_eval(s, n, sr) == v, (s, n, sr)


def test_accuracy_bound(tools_scalars):
    for e, w0, t, v in tools_scalars["accuracy_bound"]:
        assert accuracy_bound(e, w0, t) == v
    with pytest.raises(BoundInapplicableError):
        accuracy_bound(0.3, 0.2, 128.0)
    for delta in (0.01, 0.1, 1.0, 3.0):  # the corollary identity (reference test_analysis.py:101-106)
        for w0 in (1.0 / 9.0, 6.39e-3):
            assert accuracy_bound(epsilon_from_delta(delta, w0, 128.0), w0, 128.0) == pytest.approx(delta, rel=1e-12)


def test_order_comparators(tools_scalars):
    for lam, e, n in tools_scalars["chebyshev_order"]:
        assert chebyshev_order(lam, e).N0 == n
    for s, d, w0, t, n in tools_scalars["order_approx"]:
        assert order_approx(s, d, w0, t).N0 == n
    for s, d, n in tools_scalars["yang_order"]:
        assert yang_order(s, d).N0 == n
    with pytest.raises(ParameterError):
        yang_order(0.0, 1.0)
    with pytest.raises(ParameterError):
        order_approx(30.0, 1.0, 1.5, 128.0)


def test_range_kernel_and_gauss_poly(tools_scalars):
    for t, s, v in tools_scalars["range_kernel"]:
        assert float(range_kernel(t, s)) == v
    for t, tau, n, s, v in tools_scalars["gauss_poly"]:
        assert gauss_poly(t, tau, n, s) == v
    assert np.allclose(range_kernel(np.array([0.0, 10.0]), 10.0), [1.0, math.exp(-0.5)])
    with pytest.raises(ParameterError):
        gauss_poly(1.0, 1.0, 0, 30.0)
