"""Pin the CPU oracle (oracle/gpa_oracle.py) against the reference's own outputs.

The fixtures were produced by the reference package (tests/golden/make_golden.py);
the oracle must reproduce them to fp64 rounding before it is trusted as the
checker for the GPU kernels.
"""

import numpy as np
import pytest

from oracle import gpa_oracle as orc


def _taps(kind, param):
    if kind == "box":
        return orc.spatial_taps("box", half_width=int(param))
    return orc.spatial_taps("gaussian", sigma_s=float(param))


CONFIGS = ["c0", "c1", "c2", "c3", "c4"]


@pytest.mark.parametrize("name", CONFIGS)
def test_oracle_matches_reference_on_config_crops(name, golden, golden_scalars):
    c = golden_scalars["cases"][name]
    param = c["half_width"] if c["kind"] == "box" else c["sigma_s"]
    W, taps, w0 = _taps(c["kind"], param)
    assert W == c["half_width"]
    assert w0 == pytest.approx(c["w0"], rel=1e-14)
    if c["delta"] is not None:
        assert orc.order_for_delta(c["sigma_r"], c["delta"], w0) == c["order"]
    out = orc.gpa(golden[f"{name}_in"], c["kind"], W, taps, c["sigma_r"], c["order"])
    assert np.max(np.abs(out - golden[f"{name}_out"])) <= 1e-9
    exact = orc.bilateral_direct(golden[f"{name}_in"], c["kind"], W, taps, c["sigma_r"])
    assert np.max(np.abs(exact - golden[f"{name}_exact"])) <= 1e-9


ENGINE_CASES = ["impulse3", "qdegenerate5", "const_box", "const_gauss", "random64_gauss5",
                "ragged_box4", "ragged_gauss25", "shift0_gauss2", "bigwindow_gauss5",
                "row1x40_box2", "col40x1_gauss1", "sigma12_box3"]


@pytest.mark.parametrize("tag", ENGINE_CASES)
def test_oracle_matches_reference_engine_cases(tag, golden, golden_scalars):
    c = golden_scalars["cases"][tag]
    W, taps, _ = _taps(c["kind"], c["param"])
    center = c["range_spec"][1] if c["range_spec"] else 128.0
    out = orc.gpa(golden[f"{tag}_in"], c["kind"], W, taps, c["sigma_r"], c["order"], center=center)
    ref = golden[f"{tag}_out"]
    scale = max(1.0, float(np.max(np.abs(ref))))
    assert np.max(np.abs(out - ref)) <= 1e-9 * scale
    if f"{tag}_exact" in golden.files:
        exact = orc.bilateral_direct(golden[f"{tag}_in"], c["kind"], W, taps, c["sigma_r"])
        assert np.max(np.abs(exact - golden[f"{tag}_exact"])) <= 1e-9


def test_oracle_spatial_filters_match_reference(golden):
    img = golden["spatial_in"]
    for W in (1, 2, 7, 10):
        _, taps, _ = orc.spatial_taps("box", half_width=W)
        assert np.max(np.abs(orc.box_sum_filter(img, W) - golden[f"spatial_box{W}"])) <= 1e-11
    for s in (1, 3, 4):
        W, taps, _ = orc.spatial_taps("gaussian", sigma_s=float(s))
        assert np.max(np.abs(orc.separable_filter(img, taps) - golden[f"spatial_gauss{s}"])) <= 1e-11


def test_oracle_orders_match_reference(golden_scalars):
    from paper_1603_08109_b200.kernels import make_spatial_kernel  # noqa: F401  (w0 only via scalars)
    for c in golden_scalars["epsilon_from_delta"]:
        d, w0, eps = c
        assert w0 * d / (256.0 + d) == pytest.approx(eps, rel=1e-15)


def test_oracle_q_floor_case(golden):
    # order 1, sigma_r 10, 255 impulse: the reference passes some pixels through
    out = orc.gpa(golden["qdegenerate5_in"], "box", 1, np.full(3, 1 / 3), 10.0, 1)
    assert np.all(np.isfinite(out))


# ----------------------------------------------------------------------------- tools (§8(f) rows 3-4)
def test_oracle_tools_pinned(tools_golden, tools_scalars):
    from paper_1603_08109_b200 import make_spatial_kernel
    for name, c in tools_scalars["convolve_direct"].items():
        k = make_spatial_kernel(c["kind"], **({"half_width": c["param"]} if c["kind"] == "box"
                                              else {"sigma_s": c["param"]}))
        out = orc.convolve_2d(tools_golden[f"conv_{name}_in"], k.weights, k.half_width)
        assert np.array_equal(out, tools_golden[f"conv_{name}_out"]), name
    for n, s, t, v in tools_scalars["kernel_error_sup"]:
        assert orc.kernel_error_sup(n, s, t) == v, (n, s, t)
    linf, mse = orc.diff_stats(tools_golden["metric_a"], tools_golden["metric_b"])
    assert linf == tools_scalars["metrics"]["linf"]
    assert 10.0 * np.log10(mse) == tools_scalars["metrics"]["mse_db"]
    q = orc.quantize_u8(tools_golden["io_edge_in"])
    assert np.array_equal(q.ravel(), tools_golden["io_edge_pgm"][-q.size:])
