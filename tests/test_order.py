"""Host-side order selection (north-star item 4) vs the reference's pinned values."""

import math

import pytest

from paper_1603_08109_b200 import (ParameterError, chernoff_order_exhaustive, epsilon_from_delta,
                                   estimate_order, lambert_w0_series, log_chernoff,
                                   make_spatial_kernel)
from paper_1603_08109_b200.synth import CONFIGS, config_order


def test_orders_match_reference_sweep(golden_scalars):
    for sigma_r, eps, n0, method, seed in golden_scalars["orders"]:
        est = estimate_order(float(sigma_r), eps, 128.0)
        assert est.N0 == n0, (sigma_r, eps)
        assert est.method == method
        if seed is not None:
            assert est.newton_trace[0] == pytest.approx(seed, rel=1e-12)


def test_epsilon_from_delta_matches_reference(golden_scalars):
    for d, w0, eps in golden_scalars["epsilon_from_delta"]:
        assert epsilon_from_delta(d, w0, 128.0) == pytest.approx(eps, rel=1e-15)


def test_table_one_orders():
    # /root/reference/pkg/tests/test_order.py:96-100 (Table I at eps = 1e-3)
    expected = {10: 214, 15: 107, 20: 67, 25: 48, 30: 37, 35: 30, 40: 25, 45: 21, 50: 19}
    for sigma_r, n0 in expected.items():
        assert estimate_order(sigma_r, 1e-3, 128.0).N0 == n0


def test_series_seed_and_newton_trace():
    est = estimate_order(10.0, 1e-3, 128.0)
    assert math.ceil(est.newton_trace[0]) == 270
    assert est.N0 == 214 and len(est.newton_trace) == 4
    assert estimate_order(10.0, 1e-3, 128.0, newton_iters=0).N0 == 270


def test_large_sigma_fixed_order():
    assert estimate_order(70.0, 1e-3, 128.0).N0 == 10
    assert estimate_order(69.9, 1e-3, 128.0).method != "fixed_large_sigma"


def test_agrees_with_exhaustive_scan():
    for sigma_r in range(10, 70):
        for eps in (1e-1, 1e-2, 1e-3):
            lam = (128.0 / sigma_r) ** 2
            fast = estimate_order(sigma_r, eps, 128.0).N0
            assert abs(fast - chernoff_order_exhaustive(lam, eps).N0) <= 1
            assert log_chernoff(fast, lam) <= math.log(eps)


def test_lambert_series_values():
    assert lambert_w0_series(0.0) == 0.0
    assert lambert_w0_series(0.1) == pytest.approx(0.1 - 0.01 + 0.0015 - (8 / 3) * 1e-4, abs=1e-15)


def test_parameter_errors():
    with pytest.raises(ParameterError):
        estimate_order(-5.0, 0.1, 128.0)
    with pytest.raises(ParameterError):
        estimate_order(30.0, 2.0, 128.0)
    with pytest.raises(ParameterError):
        estimate_order(30.0, 0.1, 0.0)
    with pytest.raises(ParameterError):
        epsilon_from_delta(0.1, 1.5, 128.0)
    with pytest.raises(ParameterError):
        epsilon_from_delta(0.0, 0.5, 128.0)


def test_config_orders(golden_scalars):
    # N = 15 / 10 / 42 / 76 / 57
    assert [config_order(c) for c in CONFIGS] == [15, 10, 42, 76, 57]
    for name in ("c2", "c3", "c4"):
        assert config_order(name) == golden_scalars["cases"][name]["order"]


def test_epsilon_gaussian_sigma5():
    w0 = make_spatial_kernel("gaussian", sigma_s=5).w0
    assert epsilon_from_delta(0.1, w0, 128.0) == pytest.approx(2.495e-6, rel=1e-3)
