"""Host-side pieces of the drop-in API that need no GPU: kernels, ranges, argument checks."""

import math

import numpy as np
import pytest

from paper_1603_08109_b200 import (RANGE_8BIT, ParameterError, RangeSpec, RangeViolationError, as_image,
                                   center, make_spatial_kernel, uncenter, validate_range)
from paper_1603_08109_b200.engine import resolve_precision


def test_box_kernel():
    k = make_spatial_kernel("box", half_width=1)
    assert k.weights.shape == (3, 3) and np.all(k.weights == 1.0 / 9.0) and k.w0 == 1.0 / 9.0
    assert np.allclose(k.weights_1d, 1.0 / 3.0)


def test_gaussian_kernel_sigma5():
    k = make_spatial_kernel("gaussian", sigma_s=5)
    assert k.half_width == 15 and k.weights.shape == (31, 31)
    offs = np.arange(-15, 16)
    total = sum(math.exp(-(i * i + j * j) / 50.0) for i in offs for j in offs)
    assert k.w0 == pytest.approx(1.0 / total, rel=1e-12)
    assert k.weights.sum() == pytest.approx(1.0, abs=1e-12)
    assert np.allclose(np.outer(k.weights_1d, k.weights_1d), k.weights, atol=1e-15)


@pytest.mark.parametrize("sigma_s", [1.0, 1.5, 2.5, 3.0, 5.0, 8.0, 9.7])
def test_gaussian_invariants(sigma_s):
    k = make_spatial_kernel("gaussian", sigma_s=sigma_s)
    assert k.half_width == math.ceil(3 * sigma_s)
    assert abs(k.weights.sum() - 1.0) <= 1e-12
    assert np.array_equal(k.weights, k.weights.T)
    assert k.w0 == k.weights.max()


def test_kernel_errors():
    with pytest.raises(ParameterError):
        make_spatial_kernel("gaussian", sigma_s=-1)
    with pytest.raises(ParameterError):
        make_spatial_kernel("box", half_width=0)
    with pytest.raises(ParameterError):
        make_spatial_kernel("box", half_width=1.5)
    with pytest.raises(ParameterError):
        make_spatial_kernel("triangle", half_width=2)


def test_range_and_centering():
    assert np.array_equal(center(np.full((4, 4), 128.0), RANGE_8BIT), np.zeros((4, 4)))
    assert center(np.array([[0.0, 255.0]]), RANGE_8BIT).tolist() == [[-128.0, 127.0]]
    with pytest.raises(RangeViolationError, match=r"300.*row=0, col=1"):
        center(np.array([[10.0, 300.0]]), RANGE_8BIT)
    assert np.array_equal(uncenter(np.zeros((3, 3)), RANGE_8BIT), np.full((3, 3), 128.0))
    with pytest.raises(ParameterError):
        RangeSpec(half_range=0.0)
    with pytest.raises(ParameterError):
        as_image(np.array([[1.0, np.nan]]))
    with pytest.raises(ParameterError):
        as_image(np.zeros((0, 3)))
    img = np.full((3, 4), 5.0)
    img[2, 1] = -1.0
    img[2, 3] = 400.0
    with pytest.raises(RangeViolationError, match=r"sample -1.0 at pixel \(row=2, col=1\) outside \[0.0, 256.0\]"):
        validate_range(img, RANGE_8BIT)


def test_precision_rule():
    assert resolve_precision("auto", (64, 64), 30.0) == 2
    assert resolve_precision("auto", (1024, 1024), 30.0) == 1
    assert resolve_precision("auto", (1024, 1024), 12.0) == 2
    assert resolve_precision("f64", (1024, 1024), 30.0) == 2
    with pytest.raises(ParameterError):
        resolve_precision("f16", (8, 8), 30.0)
