"""GPU kernels of the tools around the filter, through the C ABI:
kernel_error_sup, image-difference metrics, convolve_direct, uint8 (PGM raster) output, the
large-window exact filter.  Checked against the reference's golden values and the oracle,
mirroring the reference's tests/test_analysis.py and tests/test_conv.py."""

import math

import numpy as np
import pytest

from oracle import gpa_oracle as orc
from paper_1603_08109_b200 import (ErrorReport, ParameterError, bilateral_exact, box_filter, convolve_direct,
                                   epsilon_from_delta, error_report, gauss_poly, gaussian_filter, gpa_filter,
                                   gpa_filter_auto, kernel_error_sup, linf_error, make_spatial_kernel, mse_db,
                                   poisson_tail, quantize, range_kernel, accuracy_bound)

pytestmark = pytest.mark.gpu

BOUND_RTOL = 1e-9


# ----------------------------------------------------------------------------- kernel_error_sup
def test_kernel_error_sup_matches_reference(tools_scalars):
    # device exp/log/lgamma vs numpy/CPython differ by ulps; the terms carry them (<= 1e-12 relative)
    for n, s, t, v in tools_scalars["kernel_error_sup"]:
        assert kernel_error_sup(n, s, t) == pytest.approx(v, rel=1e-10, abs=1e-300), (n, s, t)


@pytest.mark.parametrize("seed", range(4))
def test_kernel_error_sup_matches_oracle_seeded(seed):
    r = np.random.default_rng(seed)
    n, s, t = int(r.integers(1, 120)), float(r.uniform(10.0, 90.0)), float(r.uniform(2.0, 140.0))
    assert kernel_error_sup(n, s, t) == pytest.approx(orc.kernel_error_sup(n, s, t), rel=1e-10, abs=1e-300)


def test_kernel_error_sup_reference_properties():
    # reference tests/test_analysis.py:43-75
    assert kernel_error_sup(300, 30.0, 128.0) <= 1e-12
    sup, bound = kernel_error_sup(40, 30.0, 128.0), poisson_tail(40, (128.0 / 30.0) ** 2)
    assert bound / 100.0 <= sup <= bound * (1 + BOUND_RTOL)
    assert kernel_error_sup(1, 30.0, 128.0) == pytest.approx(1.0 - math.exp(-(128.0 ** 2) / 900.0), rel=1e-9)
    for n, s in ((40, 30), (20, 50), (10, 70), (214, 10)):
        assert kernel_error_sup(n, s, 128.0) <= poisson_tail(n, (128.0 / s) ** 2) * (1 + BOUND_RTOL)
    n, s, t = 25, 50.0, 128.0
    grid = np.arange(-int(t), int(t) + 1, 16, dtype=float)
    direct = max(abs(float(range_kernel(a - b, s)) - gauss_poly(a, b, n, s)) for a in grid for b in grid)
    sup = kernel_error_sup(n, s, t)
    assert sup * 0.5 <= direct <= sup * (1 + 1e-9)
    with pytest.raises(ParameterError):
        kernel_error_sup(0, 30.0, 128.0)
    with pytest.raises(ParameterError):
        kernel_error_sup(5, -1.0, 128.0)


# ----------------------------------------------------------------------------- metrics
def test_metrics_match_reference(tools_golden, tools_scalars):
    a, b = tools_golden["metric_a"], tools_golden["metric_b"]
    m = tools_scalars["metrics"]
    assert linf_error(a, b) == m["linf"]          # exact: same fp64 differences
    assert mse_db(a, b) == pytest.approx(m["mse_db"], abs=1e-12)
    rep = error_report(a, b)
    assert isinstance(rep, ErrorReport) and rep.linf_db == pytest.approx(m["linf_db"], abs=1e-12)


def test_metrics_reference_cases():
    # reference tests/test_analysis.py:18-40
    a = np.zeros((4, 4))
    b = a.copy()
    assert linf_error(a, b) == 0.0
    b[2, 1] += 2.0
    assert linf_error(a, b) == 2.0
    with pytest.raises(ParameterError, match="dimensions differ"):
        linf_error(np.zeros((2, 2)), np.zeros((3, 2)))
    z = np.zeros((5, 5))
    assert mse_db(z, z) == -math.inf
    assert mse_db(z, z + 1.0) == pytest.approx(0.0, abs=1e-12)
    assert mse_db(z, z + 10.0) == pytest.approx(20.0, abs=1e-12)
    rep = error_report(np.ones((3, 3)), np.ones((3, 3)))
    assert rep.linf == 0.0 and rep.linf_db == -math.inf and rep.mse_db == -math.inf


def test_metrics_checks_and_dtypes():
    a = np.arange(12.0).reshape(3, 4)
    with pytest.raises(ParameterError, match="non-finite"):
        linf_error(np.where(a > 5, np.nan, a), a)
    with pytest.raises(ParameterError, match="non-finite"):
        mse_db(a, np.where(a > 5, np.inf, a))
    with pytest.raises(ParameterError, match="non-empty 2-D"):
        linf_error(a, np.zeros(3))
    # uint8 / float32 / strided inputs read in place
    u8 = (a * 3).astype(np.uint8)
    f32 = np.asfortranarray(a.astype(np.float32))
    assert linf_error(u8, f32) == float(np.max(np.abs(u8.astype(float) - a)))


def test_metrics_on_device_tensors():
    torch = pytest.importorskip("torch")
    r = np.random.default_rng(1)
    a, b = r.uniform(0, 255, (300, 257)), r.uniform(0, 255, (300, 257))
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    linf, mse = orc.diff_stats(a, b)
    assert linf_error(ta, tb) == linf
    assert mse_db(ta, b) == pytest.approx(10.0 * math.log10(mse), abs=1e-12)


# ----------------------------------------------------------------------------- convolve_direct
def test_convolve_direct_bit_exact_vs_reference(tools_golden, tools_scalars):
    for name, c in tools_scalars["convolve_direct"].items():
        k = make_spatial_kernel(c["kind"], **({"half_width": c["param"]} if c["kind"] == "box"
                                              else {"sigma_s": c["param"]}))
        out = convolve_direct(tools_golden[f"conv_{name}_in"], k)
        assert out.dtype == np.float64 and np.array_equal(out, tools_golden[f"conv_{name}_out"]), name


@pytest.mark.parametrize("kind,param", [("box", 4), ("gaussian", 2.0), ("box", 80)])
def test_convolve_direct_vs_fast_filters(kind, param, random_image):
    # reference tests/test_conv.py: the O(1) / separable filters equal the direct sum to 1e-9
    img = random_image(170, 181)
    k = make_spatial_kernel(kind, **({"half_width": param} if kind == "box" else {"sigma_s": param}))
    direct = convolve_direct(img, k)
    assert np.array_equal(direct, orc.convolve_2d(img, k.weights, k.half_width))
    fast = box_filter(img, param) if kind == "box" else gaussian_filter(img, param)
    assert np.max(np.abs(direct - fast)) <= 1e-9


def test_convolve_direct_checks():
    k = make_spatial_kernel("gaussian", sigma_s=2.0)  # W = 6: the window check applies to Gaussians too
    with pytest.raises(ParameterError, match="too large"):
        convolve_direct(np.zeros((5, 20)), k)
    with pytest.raises(ParameterError, match="non-finite"):
        convolve_direct(np.full((20, 20), np.nan), k)
    row = np.arange(30.0)[None, :]  # 1 x N behaves as a 1-D signal
    assert np.array_equal(convolve_direct(row, k), orc.convolve_2d(row, k.weights, 6))


# ----------------------------------------------------------------------------- uint8 output
@pytest.mark.parametrize("kind,param,sr,n", [("box", 3, 30.0, 40), ("gaussian", 2.0, 50.0, 22),
                                             ("box", 20, 25.0, 57), ("gaussian", 8.0, 20.0, 76)])
@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_u8_output_is_quantised_result(kind, param, sr, n, precision, random_image):
    img = random_image(261, 307).astype(np.uint8)
    k = make_spatial_kernel(kind, **({"half_width": param} if kind == "box" else {"sigma_s": param}))
    u8 = gpa_filter(img, k, sr, n, precision=precision, out_dtype=np.uint8)
    ref = gpa_filter(img, k, sr, n, precision=precision)
    assert u8.dtype == np.uint8 and np.array_equal(u8, quantize(ref))
    assert np.array_equal(u8, orc.quantize_u8(ref))


def test_u8_output_device_tensor_and_edges(random_image):
    torch = pytest.importorskip("torch")
    k = make_spatial_kernel("box", half_width=2)
    img = random_image(67, 53)  # odd width: the packed 16-byte store falls back at the row tails
    t = torch.from_numpy(img.astype(np.uint8)).cuda()
    out = gpa_filter(t, k, 30.0, 30, out_dtype=np.uint8)
    assert out.is_cuda and out.dtype == torch.uint8
    assert np.array_equal(out.cpu().numpy(), quantize(gpa_filter(img, k, 30.0, 30)))
    # the Q-floor pass-through writes the input sample, quantised
    imp = np.zeros((3, 3))
    imp[1, 1] = 255.0
    out = gpa_filter(imp, make_spatial_kernel("box", half_width=1), 10.0, 5, out_dtype=np.uint8)
    assert np.array_equal(out, quantize(gpa_filter(imp, make_spatial_kernel("box", half_width=1), 10.0, 5)))


# ----------------------------------------------------------------------------- bounds end to end
def test_end_to_end_bound_dominates_observed_error(random_image):
    # reference tests/test_analysis.py:113-120
    img = random_image(32, 32)
    k = make_spatial_kernel("box", half_width=3)
    sigma_r, n = 30.0, 35
    fast = gpa_filter(img, k, sigma_r, n)
    exact = bilateral_exact(img, k, sigma_r)
    assert linf_error(fast, exact) <= accuracy_bound(kernel_error_sup(n, sigma_r, 128.0), k.w0, 128.0)


def test_auto_error_below_delta(random_image):
    img = random_image(32, 32)
    k = make_spatial_kernel("gaussian", sigma_s=3)
    fast, est = gpa_filter_auto(img, k, 50.0, 0.1)
    assert linf_error(fast, bilateral_exact(img, k, 50.0)) <= 0.1
    assert est.epsilon == epsilon_from_delta(0.1, k.w0, 128.0)


def test_bilateral_exact_large_window(random_image):
    # W > 77 runs the untiled variant (the (16 + 2W)^2 tile exceeds shared memory)
    img = random_image(170, 175)
    k = make_spatial_kernel("box", half_width=80)
    out = bilateral_exact(img, k, 30.0)
    ref = orc.bilateral_direct(img, "box", 80, k.weights_1d, 30.0)
    assert np.max(np.abs(out - ref)) <= 1e-9  # 161^2 = 25,921 summed terms per pixel
