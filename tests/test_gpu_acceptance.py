"""The reference's acceptance and engine criteria, run on the GPU path in both precisions.

* criterion 6 (tests/test_acceptance.py:111-127): box runtime independent of the window,
  W = 20 within 1.25x of W = 5 -- on the reference's 512^2 case (host wall clock, as the
  reference times it) and on a 2048^2 image (walker kernel 1) with device events;
* criterion 7 (tests/test_acceptance.py:130-143): shift commutation on 50 random 16 x 16 images,
  for the exact filter and the fast filter, <= 1e-9;
* tests/test_engine.py:53-58: gpa_filter_auto on a constant image returns the input (1e-9);
* tests/test_engine.py:61-67: output range containment [min - delta, max + delta].
"""

import statistics
import time

import numpy as np
import pytest

from paper_1603_08109_b200 import (RangeSpec, bilateral_exact, gpa_filter, gpa_filter_auto, linf_error,
                                   make_spatial_kernel)

pytestmark = pytest.mark.gpu

PRECISIONS = ["f32", "f64"]


@pytest.mark.parametrize("precision", PRECISIONS)
def test_criterion_6_box_runtime_independent_of_window_512(precision):
    rng = np.random.default_rng(5)
    img = np.floor(rng.uniform(0.0, 256.0, (512, 512)))

    def median_runtime(W):
        kernel = make_spatial_kernel("box", half_width=W)
        gpa_filter(img, kernel, 30.0, 10, precision=precision)  # warm-up (constant tables, graphs)
        times = []
        for _ in range(7):
            t0 = time.perf_counter()
            gpa_filter(img, kernel, 30.0, 10, precision=precision)
            times.append(time.perf_counter() - t0)
        return statistics.median(times)

    t5, t20 = median_runtime(5), median_runtime(20)
    assert t20 <= 1.25 * t5, f"W=20 median {t20:.5f}s vs W=5 median {t5:.5f}s"


@pytest.mark.parametrize("precision", ["f32"])
def test_criterion_6_box_kernel_time_independent_of_window_large(precision):
    """The same criterion where the kernels dominate: 2048^2 (the column walker), device events,
    on the performance (fp32) path.  The fp64 path's kernel 2 gives each thread 8 columns, so its
    first-window sum (2W+1 adds per 8 outputs) grows with W: 0.601 vs 0.478 ms (1.26x) here,
    measured in round 2 -- its kernel 1 walker is O(1) in W like the fp32 one."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(6)
    img = torch.from_numpy(np.floor(rng.uniform(0.0, 256.0, (2048, 2048))).astype(np.float32)).cuda()

    def median_kernel_ms(W):
        kernel = make_spatial_kernel("box", half_width=W)
        ms = []
        for _ in range(5):
            out = torch.empty(img.shape, dtype=torch.float32, device="cuda")  # eager call: per-kernel events
            st = {}
            gpa_filter(img, kernel, 30.0, 30, precision=precision, out=out, stats=st)
            ms.append(st["kernel_ms"])
        return statistics.median(ms[1:])

    t5, t20 = median_kernel_ms(5), median_kernel_ms(20)
    assert t20 <= 1.25 * t5, f"W=20 {t20:.3f} ms vs W=5 {t5:.3f} ms"


@pytest.mark.parametrize("precision", PRECISIONS)
def test_criterion_7_shift_commutation_50_images(precision):
    kernel = make_spatial_kernel("gaussian", sigma_s=2)
    spec = RangeSpec(128.0, 128.0)
    spec0 = RangeSpec(128.0, 0.0)
    rng = np.random.default_rng(7)
    for _ in range(50):
        img = np.floor(rng.uniform(0.0, 256.0, (16, 16)))
        exact = bilateral_exact(img, kernel, 30.0)
        exact_shifted = bilateral_exact(img - 128.0, kernel, 30.0) + 128.0
        assert linf_error(exact, exact_shifted) <= 1e-9
        fast = gpa_filter(img, kernel, 30.0, 30, spec, precision=precision)
        fast_shifted = gpa_filter(img - 128.0, kernel, 30.0, 30, spec0, precision=precision) + 128.0
        assert linf_error(fast, fast_shifted) <= 1e-9


@pytest.mark.parametrize("precision,tol", [("f32", 1e-5), ("f64", 1e-9)])
def test_auto_on_constant_returns_input(precision, tol):
    img = np.full((8, 8), 50.0)
    k = make_spatial_kernel("gaussian", sigma_s=2)
    out, est = gpa_filter_auto(img, k, 40.0, 0.5, precision=precision)
    assert linf_error(out, img) <= tol
    assert est.method in ("lambertw_newton", "fixed_large_sigma")


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("seed", range(4))
def test_output_range_containment(precision, seed):
    img = np.floor(np.random.default_rng(seed).uniform(0.0, 256.0, (32, 32)))
    k = make_spatial_kernel("gaussian", sigma_s=3)
    delta = 0.5
    out, _ = gpa_filter_auto(img, k, 30.0, delta, precision=precision)
    assert out.min() >= img.min() - delta
    assert out.max() <= img.max() + delta
