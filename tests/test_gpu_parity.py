"""GPU parity: the CUDA path (through the C ABI) vs the reference's golden outputs and the oracle.

Tolerances: fp64 path <= 1e-9 gray levels (scale-relative for large values);
fp32 path <= 1e-3 gray levels, the north-star bar (max |delta| vs the
reference's float64 output on identical inputs).
"""

import numpy as np
import pytest

from oracle import gpa_oracle as orc
from paper_1603_08109_b200 import (NumericRangeError, ParameterError, RangeSpec, RangeViolationError,
                                   apply_spatial, box_filter, gaussian_filter, gpa_filter, gpa_filter_auto,
                                   make_spatial_kernel, synth)
from paper_1603_08109_b200 import _native

pytestmark = pytest.mark.gpu

F32_TOL = 1e-3
F64_TOL = 1e-9


def kern(kind, param):
    return (make_spatial_kernel("box", half_width=int(param)) if kind == "box"
            else make_spatial_kernel("gaussian", sigma_s=float(param)))


def oracle(img, k, sigma_r, N, center=128.0):
    return orc.gpa(img, k.kind, k.half_width, k.weights_1d, sigma_r, N, center=center)


# ----------------------------------------------------------------------------- golden
ENGINE_CASES = ["impulse3", "qdegenerate5", "const_box", "const_gauss", "random64_gauss5",
                "ragged_box4", "ragged_gauss25", "shift0_gauss2", "bigwindow_gauss5",
                "row1x40_box2", "col40x1_gauss1", "sigma12_box3"]


@pytest.mark.parametrize("tag", ENGINE_CASES)
def test_reference_engine_cases_fp64(tag, golden, golden_scalars):
    c = golden_scalars["cases"][tag]
    k = kern(c["kind"], c["param"])
    spec = RangeSpec(*c["range_spec"]) if c["range_spec"] else None
    stats = {}
    out = gpa_filter(golden[f"{tag}_in"], k, c["sigma_r"], c["order"], spec,
                     allow_small_sigma=c["allow_small_sigma"], stats=stats)
    ref = golden[f"{tag}_out"]
    assert out.dtype == np.float64 and out.shape == ref.shape
    assert stats["spatial_filter_calls"] == c["order"] + 1 and stats["precision"] == "f64"
    scale = max(1.0, float(np.max(np.abs(ref))))
    assert np.max(np.abs(out - ref)) <= F64_TOL * scale, tag


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "c4"])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_reference_config_crops(name, precision, golden, golden_scalars):
    c = golden_scalars["cases"][name]
    k = kern(c["kind"], c["half_width"] if c["kind"] == "box" else c["sigma_s"])
    img = golden[f"{name}_in"]
    if c["delta"] is not None:
        out, est = gpa_filter_auto(img, k, c["sigma_r"], c["delta"], precision=precision)
        assert est.N0 == c["order"]
    else:
        out = gpa_filter(img, k, c["sigma_r"], c["order"], precision=precision)
    err = np.max(np.abs(out - golden[f"{name}_out"]))
    assert err <= (F64_TOL if precision == "f64" else F32_TOL), err


@pytest.mark.parametrize("tag", ["c0", "c1", "c2", "c3", "c4", "impulse3", "random64_gauss5", "ragged_box4",
                                 "ragged_gauss25", "shift0_gauss2"])
def test_bilateral_exact_matches_reference(tag, golden, golden_scalars):
    """GPU brute force (fp64) = the reference's bilateral_exact (reference.py:17-45) outputs."""
    from paper_1603_08109_b200 import bilateral_exact
    c = golden_scalars["cases"][tag]
    if "half_width" in c:
        k = kern(c["kind"], c["half_width"] if c["kind"] == "box" else c["sigma_s"])
    else:
        k = kern(c["kind"], c["param"])
    out = bilateral_exact(golden[f"{tag}_in"], k, c["sigma_r"])
    assert np.max(np.abs(out - golden[f"{tag}_exact"])) <= 1e-10


def test_bilateral_exact_errors():
    from paper_1603_08109_b200 import bilateral_exact
    k = make_spatial_kernel("box", half_width=1)
    img = np.floor(np.random.default_rng(2).uniform(0, 256, (8, 8)))
    with pytest.raises(ParameterError):
        bilateral_exact(img, k, -1.0)
    with pytest.raises(ParameterError):
        bilateral_exact(img, make_spatial_kernel("box", half_width=8), 30.0)


def test_spatial_filters_match_reference(golden):
    img = golden["spatial_in"]
    for W in (1, 2, 7, 10):
        assert np.max(np.abs(box_filter(img, W) - golden[f"spatial_box{W}"])) <= 1e-11
    for s in (1, 3, 4):
        assert np.max(np.abs(gaussian_filter(img, float(s)) - golden[f"spatial_gauss{s}"])) <= 1e-11
        k = make_spatial_kernel("gaussian", sigma_s=float(s))
        assert np.max(np.abs(apply_spatial(img, k) - golden[f"spatial_gauss{s}"])) <= 1e-11


# ----------------------------------------------------------------------------- seeded sweeps vs oracle
SWEEP = [
    # (h, w, kind, param, sigma_r, N)
    (1, 37, "box", 2, 30.0, 12),
    (29, 1, "gaussian", 1.0, 30.0, 12),
    (2, 2, "gaussian", 3.0, 40.0, 10),
    (70, 131, "box", 1, 50.0, 10),
    (97, 65, "box", 5, 30.0, 30),
    (130, 200, "box", 20, 25.0, 57),
    (64, 300, "gaussian", 2.0, 20.0, 40),
    (200, 130, "gaussian", 3.0, 40.0, 15),
    (160, 170, "gaussian", 5.0, 30.0, 42),
    (130, 140, "gaussian", 8.0, 20.0, 76),
    (90, 90, "gaussian", 12.0, 35.0, 30),
]


@pytest.mark.parametrize("h,w,kind,param,sigma_r,N", SWEEP)
@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_sweep_vs_oracle(h, w, kind, param, sigma_r, N, precision):
    rng = np.random.default_rng(h * 1000 + w)
    img = np.floor(rng.uniform(0.0, 256.0, (h, w)))
    k = kern(kind, param)
    if kind == "box" and param >= min([d for d in (h, w) if d > 1], default=1):
        pytest.skip("window too large")
    out = gpa_filter(img, k, sigma_r, N, precision=precision)
    ref = oracle(img, k, sigma_r, N)
    err = np.max(np.abs(out - ref))
    assert err <= (1e-8 if precision == "f64" else F32_TOL), err


@pytest.mark.parametrize("dtype", [np.uint8, np.float32, np.float64])
def test_input_dtypes_agree(dtype):
    rng = np.random.default_rng(11)
    img = np.floor(rng.uniform(0.0, 256.0, (300, 260))).astype(dtype)
    k = make_spatial_kernel("gaussian", sigma_s=3.0)
    out = gpa_filter(img, k, 40.0, 15)
    ref = gpa_filter(img.astype(np.float64), k, 40.0, 15)
    assert np.array_equal(out, ref)


def test_strided_input():
    rng = np.random.default_rng(12)
    big = np.floor(rng.uniform(0.0, 256.0, (300, 400)))
    view = big[10:260, 20:330]
    k = make_spatial_kernel("box", half_width=4)
    assert np.array_equal(gpa_filter(view, k, 30.0, 20), gpa_filter(view.copy(), k, 30.0, 20))


def test_row_bands_bit_exact():
    """Splitting into row bands (workspace limit) must not change a single bit."""
    rng = np.random.default_rng(13)
    img = np.floor(rng.uniform(0.0, 256.0, (517, 300)))
    for k, N in ((make_spatial_kernel("box", half_width=7), 20), (make_spatial_kernel("gaussian", sigma_s=4), 30)):
        s1, s2 = {}, {}
        full = gpa_filter(img, k, 30.0, N, precision="f32", stats=s1)
        _native.set_workspace_limit(1 << 20)
        try:
            banded = gpa_filter(img, k, 30.0, N, precision="f32", stats=s2)
        finally:
            _native.set_workspace_limit(8 << 30)
        assert s1["bands"] == 1 and s2["bands"] > 1
        assert np.array_equal(full, banded)


def test_batch_matches_single_and_names_bad_image():
    from paper_1603_08109_b200 import gpa_filter_batch
    rng = np.random.default_rng(21)
    imgs = [np.floor(rng.uniform(0.0, 256.0, (h, 260))).astype(np.float32) for h in (300, 257, 64, 300)]
    k = make_spatial_kernel("gaussian", sigma_s=3.0)
    stats = {}
    outs = gpa_filter_batch(imgs, k, 40.0, 15, stats=stats, precision="f32")
    assert stats["launches"] == len(imgs)  # small images: one fused kernel each (fb_small.cuh)
    for im, o in zip(imgs, outs):
        assert np.array_equal(o, gpa_filter(im, k, 40.0, 15, precision="f32"))
    bad = [im.copy() for im in imgs]
    bad[2][5, 7] = 300.0
    with pytest.raises(RangeViolationError, match=r"row=5, col=7"):
        gpa_filter_batch(bad, k, 40.0, 15, precision="f32")


def test_chunked_host_pipeline_matches_device_path():
    """Host images > 4 MP are pipelined in row chunks (multiples of 256 rows) over three streams.
    The box walks start at image rows that are multiples of 256 whatever the chunking, so the
    chunked host path is bit-identical to one device-resident call; both are also checked against
    the fp64 path (itself pinned to the reference at 1e-9)."""
    torch = pytest.importorskip("torch")
    cfg = synth.CONFIGS["c4"]
    img = synth.config_image(cfg, height=2304, width=2048)
    for k, N in ((synth.config_kernel(cfg), 57), (make_spatial_kernel("gaussian", sigma_s=5.0), 42)):
        stats = {}
        host = gpa_filter(img, k, 25.0, N, precision="f32", stats=stats)
        assert stats["h2d_bytes"] == img.nbytes and stats["d2h_bytes"] == host.nbytes
        dev = gpa_filter(torch.from_numpy(img).cuda(), k, 25.0, N, precision="f32").cpu().numpy()
        ref = gpa_filter(img, k, 25.0, N, precision="f64")
        assert np.array_equal(host, dev)
        assert np.max(np.abs(dev - ref)) <= 5e-4


def test_cuda_tensor_in_tensor_out():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(14)
    img = np.floor(rng.uniform(0.0, 256.0, (257, 301))).astype(np.float32)
    k = make_spatial_kernel("gaussian", sigma_s=2.0)
    host = gpa_filter(img, k, 30.0, 20)
    dev = gpa_filter(torch.from_numpy(img).cuda(), k, 30.0, 20)
    assert dev.is_cuda and dev.dtype == torch.float64
    assert np.array_equal(dev.cpu().numpy(), host)
    dev32 = gpa_filter(torch.from_numpy(img).cuda(), k, 30.0, 20, out_dtype=np.float32)
    assert dev32.dtype == torch.float32
    assert np.max(np.abs(dev32.cpu().numpy() - host)) <= 1e-4


# ----------------------------------------------------------------------------- reference engine tests
def test_constant_passthrough_any_precision():
    # reference bar 1e-9 (test_engine.py:9-14) holds in fp64; fp32 channels round at ~1e-7 relative
    img = np.full((300, 300), 93.0)
    for k in (make_spatial_kernel("box", half_width=3), make_spatial_kernel("gaussian", sigma_s=2)):
        for prec, tol in (("f32", 1e-5), ("f64", 1e-9)):
            assert np.max(np.abs(gpa_filter(img, k, 40.0, 25, precision=prec) - img)) <= tol


def test_shift_commutation_fp32():
    k = make_spatial_kernel("gaussian", sigma_s=2)
    rng = np.random.default_rng(15)
    img = np.floor(rng.uniform(0.0, 256.0, (300, 280)))
    direct = gpa_filter(img, k, 30.0, 40, RangeSpec(128.0, 128.0), precision="f32")
    shifted = gpa_filter(img - 128.0, k, 30.0, 40, RangeSpec(128.0, 0.0), precision="f32") + 128.0
    assert np.max(np.abs(direct - shifted)) <= 1e-9


def test_delta_guarantee_vs_brute_force():
    rng = np.random.default_rng(20240817)
    img = np.floor(rng.uniform(0.0, 256.0, (64, 64)))
    for k in (make_spatial_kernel("gaussian", sigma_s=3), make_spatial_kernel("box", half_width=4),
              make_spatial_kernel("box", half_width=10)):
        for sigma_r in (30.0, 50.0):
            exact = orc.bilateral_direct(img, k.kind, k.half_width, k.weights_1d, sigma_r)
            for delta in (0.1, 1.0):
                for prec in ("f32", "f64"):
                    fast, _ = gpa_filter_auto(img, k, sigma_r, delta, precision=prec)
                    assert np.max(np.abs(fast - exact)) <= delta


def test_monotone_error_decay():
    rng = np.random.default_rng(8)
    img = np.floor(rng.uniform(0.0, 256.0, (64, 64)))
    k = make_spatial_kernel("gaussian", sigma_s=5)
    exact = orc.bilateral_direct(img, k.kind, k.half_width, k.weights_1d, 30.0)
    errs = [np.max(np.abs(gpa_filter(img, k, 30.0, n) - exact)) for n in (10, 20, 30, 40, 50, 60)]
    assert all(a >= b for a, b in zip(errs, errs[1:])), errs
    assert errs[0] >= 10.0 * errs[3]


def test_errors_and_precedence():
    k = make_spatial_kernel("box", half_width=1)
    img = np.floor(np.random.default_rng(1).uniform(0, 256, (8, 8)))
    bad = img.copy()
    bad[3, 5] = 400.0
    bad[6, 1] = -2.0
    with pytest.raises(RangeViolationError, match=r"sample 400.0 at pixel \(row=3, col=5\) outside \[0.0, 256.0\]"):
        gpa_filter(bad, k, 30.0, 10)
    # input errors win over parameter errors (image validated first, engine.py:36-49)
    with pytest.raises(RangeViolationError):
        gpa_filter(bad, k, -1.0, 10)
    nan = img.copy()
    nan[2, 2] = np.nan
    with pytest.raises(ParameterError, match="non-finite"):
        gpa_filter(nan, k, 30.0, 10)
    with pytest.raises(ParameterError):
        gpa_filter(img, k, 5.0, 10)
    with pytest.raises(ParameterError):
        gpa_filter(img, k, 30.0, 0)
    with pytest.raises(ParameterError):
        gpa_filter(img, k, 30.0, 2.5)
    with pytest.raises(ParameterError, match="too large"):
        gpa_filter(img, make_spatial_kernel("box", half_width=8), 30.0, 10)
    with pytest.raises(ParameterError):
        gpa_filter(np.zeros((0, 4)), k, 30.0, 10)
    with pytest.raises(ParameterError):
        gpa_filter(np.zeros((4, 4, 1)), k, 30.0, 10)
    with pytest.raises(ParameterError):
        box_filter(np.zeros((8, 20)), 8)
    # the override runs: finite output or NumericRangeError, never silent corruption
    try:
        out = gpa_filter(img, k, 9.0, 300, allow_small_sigma=True)
        assert np.all(np.isfinite(out))
    except NumericRangeError:
        pass


def test_q_degeneracy_falls_back_to_input(golden):
    img = np.zeros((5, 5))
    img[2, 2] = 255.0
    stats = {}
    out = gpa_filter(img, make_spatial_kernel("box", half_width=1), 10.0, 1, allow_small_sigma=True, stats=stats)
    assert np.all(np.isfinite(out))
    assert np.array_equal(out, golden["qdegenerate5_out"])


# ----------------------------------------------------------------------------- full-size locality checks
def _window_check(img, out, k, sigma_r, N, windows, tol):
    """The filter is local (radius W, replicate boundary): the oracle on a window plus a W margin
    reproduces the interior exactly, so full-size outputs can be checked window by window."""
    W = k.half_width
    H, Wd = img.shape
    worst = 0.0
    for (y, x, h, w) in windows:
        y0, x0 = max(0, y - W), max(0, x - W)
        y1, x1 = min(H, y + h + W), min(Wd, x + w + W)
        sub = oracle(img[y0:y1, x0:x1], k, sigma_r, N)
        ref = sub[y - y0:y - y0 + h, x - x0:x - x0 + w]
        worst = max(worst, float(np.max(np.abs(out[y:y + h, x:x + w] - ref))))
    assert worst <= tol, worst
    return worst


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3"])
def test_full_size_config_windows(name):
    cfg = synth.CONFIGS[name]
    img = synth.config_image(cfg)
    k = synth.config_kernel(cfg)
    N = synth.config_order(cfg)
    out = gpa_filter(img, k, cfg.sigma_r, N)
    H, Wd = img.shape
    windows = [(0, 0, 48, 48), (H - 48, Wd - 48, 48, 48), (H // 2, Wd // 3, 64, 64), (0, Wd // 2, 40, 64),
               (H // 3, 0, 64, 40)]
    _window_check(img, out, k, cfg.sigma_r, N, windows, F32_TOL)


@pytest.mark.slow
def test_full_size_c4_windows():
    cfg = synth.CONFIGS["c4"]
    img = synth.config_image(cfg)
    k = synth.config_kernel(cfg)
    N = synth.config_order(cfg)
    out = gpa_filter(img, k, cfg.sigma_r, N, out_dtype=np.float32)
    H, Wd = img.shape
    windows = [(0, 0, 48, 48), (H - 48, Wd - 48, 48, 48), (H // 2 + 5, Wd // 3 + 7, 64, 64),
               (8191, 8100, 40, 40), (H - 30, 0, 30, 64)]
    _window_check(img, out.astype(np.float64), k, cfg.sigma_r, N, windows, F32_TOL)


def test_default_stream_work_is_ordered_before_the_call():
    """A tensor still being written by torch on the legacy default stream is read only after that
    write (fb_set_stream(cudaStreamLegacy): the context's stream waits for it at every call)."""
    torch = pytest.importorskip("torch")
    x = torch.zeros((1024, 1024), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    k = make_spatial_kernel("box", half_width=5)
    for _ in range(3):
        torch.cuda._sleep(100_000_000)  # ~50 ms spin on the default stream, then the write
        x.fill_(200.0)
        out = gpa_filter(x, k, 50.0, 10, precision="f32").cpu().numpy()
        assert np.max(np.abs(out - 200.0)) <= 1e-4
        x.zero_()


def test_concurrent_calls_from_threads():
    """ctypes releases the GIL: calls from several host threads share one device context, which
    the binding serialises (a context is not re-entrant)."""
    import threading
    rng = np.random.default_rng(7)
    imgs = [np.floor(rng.uniform(0, 256, (300 + 17 * i, 257))).astype(np.float32) for i in range(6)]
    k = make_spatial_kernel("gaussian", sigma_s=3.0)
    want = [gpa_filter(im, k, 40.0, 15, precision="f32") for im in imgs]
    got = [None] * len(imgs)

    def work(i):
        for _ in range(5):
            got[i] = gpa_filter(imgs[i], k, 40.0, 15, precision="f32")

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(imgs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for w, g in zip(want, got):
        assert np.array_equal(w, g)
