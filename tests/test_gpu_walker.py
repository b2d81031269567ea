"""GPU parity of the large-image box path (kernel 1 = the column walker with TMA row stores,
kernel 2 = the fast horizontal pass + fp64 Horner; and the fp64 walker / kernel 2 of
fb_fast64.cuh) and of kernel 2's epilogue paths.

The walker runs when (cols + 2W) x image rows >= 4 Mi samples and N+1 <= 64, so these images are
~2100^2.  Full images are compared with the fp64 path (pinned to the reference at 1e-9 by
test_gpu_parity.py); windows are compared with the oracle itself.
"""

import numpy as np
import pytest

from oracle import gpa_oracle as orc
from paper_1603_08109_b200 import _native, gpa_filter, make_spatial_kernel, synth

pytestmark = pytest.mark.gpu

F32_TOL = 1e-3
SIDE = 2100  # (2100 + 2W) * 2100 >= 4 Mi: walker territory


def _windows(H, Wd):
    return [(0, 0, 40, 40), (H - 40, Wd - 40, 40, 40), (H // 2 + 3, Wd // 3 + 5, 48, 48), (0, Wd - 40, 40, 40)]


def _oracle_windows(img, out, k, sigma_r, N):
    W = k.half_width
    H, Wd = img.shape
    worst = 0.0
    for (y, x, h, w) in _windows(H, Wd):
        y0, x0 = max(0, y - W), max(0, x - W)
        y1, x1 = min(H, y + h + W), min(Wd, x + w + W)
        sub = orc.gpa(img[y0:y1, x0:x1].astype(np.float64), "box", W, k.weights_1d, sigma_r, N)
        ref = sub[y - y0:y - y0 + h, x - x0:x - x0 + w]
        worst = max(worst, float(np.max(np.abs(out[y:y + h, x:x + w] - ref))))
    return worst


# Orders are in the convergent regime of each sigma_r (Algorithm 1 at delta = 1 gives >= these;
# N = 7 at sigma_r = 400 covers the smallest channel capacity, which Algorithm 1's floor of 10
# never selects).  Far below Algorithm 1's order the truncated series itself is meaningless
# (outputs of 1e6 gray levels) and no fp32 bar applies.
@pytest.mark.parametrize("W,N,sigma_r,dtype", [
    (1, 7, 400.0, np.float32),    # NCH 8
    (1, 49, 25.0, np.float32),    # smallest window at its Algorithm-1 order (delta = 1)
    (5, 10, 150.0, np.float32),   # NCH 16, N+1 just past a multiple of 8
    (3, 28, 40.0, np.uint8),      # register-path input (no cp.async ring)
    (20, 57, 25.0, np.float32),   # c4's filter
    (20, 57, 25.0, np.float64),
    (32, 63, 23.5, np.float32),   # NCH 64 = the walker's capacity, widest fast window
])
def test_walker_matches_oracle_and_fp64(W, N, sigma_r, dtype):
    img = synth.config_image("c4", height=SIDE, width=SIDE)  # c4 recipe: outliers included
    img = np.floor(img).astype(dtype)
    k = make_spatial_kernel("box", half_width=W)
    out = gpa_filter(img, k, sigma_r, N, precision="f32")
    ref64 = gpa_filter(img, k, sigma_r, N, precision="f64")
    assert np.max(np.abs(out - ref64)) <= 5e-4
    assert _oracle_windows(img, out, k, sigma_r, N) <= F32_TOL
    # the fp64 path at this size runs its own walker (fb_fast64.cuh): oracle-exact
    assert _oracle_windows(img, ref64, k, sigma_r, N) <= 1e-8


def test_fp64_walker_bands_and_halos_are_exact():
    """The fp64 walker (fb_fast64.cuh) is partition-independent: two bands and a band call with
    separate halo buffers reproduce the single call bit for bit."""
    torch = pytest.importorskip("torch")
    img = synth.config_image("c4", height=4096, width=2048)
    k = make_spatial_kernel("box", half_width=20)
    N, W = 57, 20
    dimg = torch.from_numpy(img).cuda()
    full = gpa_filter(dimg, k, 25.0, N, precision="f64").cpu().numpy()
    pitch = (2048 + 40 + 31) // 32 * 32
    _native.set_workspace_limit(2048 * (N + 1) * pitch * 8)
    try:
        st = {}
        banded = gpa_filter(dimg, k, 25.0, N, precision="f64", stats=st).cpu().numpy()
    finally:
        _native.set_workspace_limit(8 << 30)
    assert st["bands"] == 2
    assert np.array_equal(banded, full)
    r0, r1 = 1024, 3100
    band = torch.from_numpy(np.ascontiguousarray(img[r0:r1])).cuda()
    above = torch.from_numpy(np.ascontiguousarray(img[r0 - W:r0])).cuda()
    below = torch.from_numpy(np.ascontiguousarray(img[r1:r1 + W])).cuda()
    out = torch.empty((r1 - r0, img.shape[1]), dtype=torch.float64, device="cuda")
    _native.gpa_band(band, out, k, 25.0, N, 128.0, 128.0, _native.FB_PREC_F64, r0, 4096, above, below, 0)
    assert np.array_equal(out.cpu().numpy(), full[r0:r1])


def test_walker_band_partitions_agree():
    """Several walker bands (workspace limit) and band calls with separate halo buffers are
    bit-identical to one band (results independent of the parallel decomposition)."""
    torch = pytest.importorskip("torch")
    img = synth.config_image("c4", height=4096, width=2048)
    k = make_spatial_kernel("box", half_width=20)
    N = 57
    one, many = {}, {}
    dimg = torch.from_numpy(img).cuda()  # device-resident: no host row chunks
    full = gpa_filter(dimg, k, 25.0, N, precision="f32", stats=one).cpu().numpy()
    pitch = (2048 + 40 + 31) // 32 * 32
    _native.set_workspace_limit(2048 * (N + 1) * pitch * 4)  # two bands of 2048 rows
    try:
        banded = gpa_filter(dimg, k, 25.0, N, precision="f32", stats=many).cpu().numpy()
    finally:
        _native.set_workspace_limit(8 << 30)
    assert one["bands"] == 1 and many["bands"] == 2
    ref64 = gpa_filter(img, k, 25.0, N, precision="f64")
    assert np.max(np.abs(full - ref64)) <= 5e-4
    assert np.array_equal(banded, full)  # walks start at image rows = multiples of 256 in both
    H, W = img.shape[0], 20
    # rows [1024, 3100) from buffers holding only those rows, and W halo rows each side in separate
    # buffers (a rank's band and its neighbours' rows, fb_gpa_filter_band): the same bits
    for r0, r1, top in ((1024, 3100, W), (0, 1280, 0), (2816, H, W), (1000, 3100, W + 1000 % 256)):
        band = torch.from_numpy(np.ascontiguousarray(img[r0:r1])).cuda()
        above = torch.from_numpy(np.ascontiguousarray(img[r0 - top:r0])).cuda() if top else None
        below = torch.from_numpy(np.ascontiguousarray(img[r1:r1 + W])).cuda() if r1 < H else None
        out = torch.empty((r1 - r0, img.shape[1]), dtype=torch.float64, device="cuda")
        _native.gpa_band(band, out, k, 25.0, N, 128.0, 128.0, _native.FB_PREC_F32, r0, H, above, below, 0)
        assert np.array_equal(out.cpu().numpy(), full[r0:r1]), (r0, r1)
    # a band off the 256-row grid with only W halo rows: its first walk re-reads rows it does not
    # have (replicated), so the bits differ -- still the same filter to fp32 rounding
    r0, r1 = 1000, 3100
    ext = torch.from_numpy(np.ascontiguousarray(img[r0 - W:r1 + W])).cuda()
    out = torch.empty((r1 - r0, img.shape[1]), dtype=torch.float32, device="cuda")
    _native.gpa(ext, out, k, 25.0, N, 128.0, 128.0, _native.FB_PREC_F32, 0, halo_top=W, halo_bottom=W)
    assert np.max(np.abs(out.cpu().numpy() - ref64[r0:r1])) <= 5e-4


def test_host_band_with_halos_chunked():
    """The multi-GPU e2e leg: a host-resident band with its halo rows in the same buffer
    (fb_gpa_filter_band with adjacent halos), pipelined in row chunks (H2D / kernels / D2H on three
    streams), is bit-identical to the same rows of the whole image."""
    img = synth.config_image("c4", height=4096, width=2048)
    k = make_spatial_kernel("box", half_width=20)
    N, W = 57, 20
    full = gpa_filter(img, k, 25.0, N, precision="f32")
    for r0, r1 in ((0, 2304), (1024, 3328), (1792, 4096)):
        top, bottom = min(W, r0), min(W, 4096 - r1)
        ext = np.ascontiguousarray(img[r0 - top:r1 + bottom])
        out = np.empty((r1 - r0, img.shape[1]), dtype=np.float64)
        st = _native.gpa_band(ext[top:top + r1 - r0], out, k, 25.0, N, 128.0, 128.0, _native.FB_PREC_F32, r0,
                              4096, ext[:top] if top else None, ext[top + r1 - r0:] if bottom else None, 0)
        assert st["h2d_bytes"] == ext.nbytes and st["d2h_bytes"] == out.nbytes
        assert np.array_equal(out, full[r0:r1]), (r0, r1)


@pytest.mark.parametrize("width", [128, 130, 131, 133, 1029])
def test_fp32_output_vector_and_scalar_stores(width):
    """float32 outputs use 128-bit stores where the row segment is aligned and complete, scalar
    stores elsewhere (odd widths, ragged right edge): both must hold the same values."""
    rng = np.random.default_rng(width)
    img = np.floor(rng.uniform(0.0, 256.0, (70, width)))
    for k, N in ((make_spatial_kernel("box", half_width=5), 20), (make_spatial_kernel("gaussian", sigma_s=3.0), 15)):
        o32 = gpa_filter(img, k, 30.0, N, precision="f32", out_dtype=np.float32)
        o64 = gpa_filter(img, k, 30.0, N, precision="f32")
        assert o32.dtype == np.float32
        assert np.array_equal(o32, o64.astype(np.float32))
        ref = orc.gpa(img, k.kind, k.half_width, k.weights_1d, 30.0, N)
        assert np.max(np.abs(o64 - ref)) <= F32_TOL


def test_fast_path_q_floor_passthrough(golden):
    """The fp32 kernels' epilogue applies the reference's |Q| < 1e-30 pass-through
    (engine.py:20, 68) like the fp64 path: same pixels, same values."""
    img = np.zeros((5, 5))
    img[2, 2] = 255.0
    k = make_spatial_kernel("box", half_width=1)
    s32, s64 = {}, {}
    o32 = gpa_filter(img, k, 10.0, 1, allow_small_sigma=True, precision="f32", stats=s32)
    o64 = gpa_filter(img, k, 10.0, 1, allow_small_sigma=True, precision="f64", stats=s64)
    assert s64["degenerate_pixels"] > 0
    assert s32["degenerate_pixels"] == s64["degenerate_pixels"]
    assert np.max(np.abs(o32 - golden["qdegenerate5_out"])) <= F32_TOL
    assert np.max(np.abs(o64 - golden["qdegenerate5_out"])) <= 1e-9


@pytest.mark.parametrize("kind,param,N", [("gaussian", 5.0, 42), ("gaussian", 8.0, 60), ("box", 20, 57)])
def test_fp64_fast_kernels_match_oracle_windows(kind, param, N):
    """precision="f64" on a large image runs the specialised fp64 kernels (fb_fast64.cuh):
    the reference's fp64 arithmetic to 1e-8 gray levels."""
    img = synth.config_image("c2", height=1200, width=1100)
    k = (make_spatial_kernel("box", half_width=int(param)) if kind == "box"
         else make_spatial_kernel("gaussian", sigma_s=param))
    sigma_r = 12.0  # below the fp32 floor: the "auto" policy's fp64 regime
    out = gpa_filter(img, k, sigma_r, N, allow_small_sigma=True)  # auto -> f64
    W = k.half_width
    H, Wd = img.shape
    worst = 0.0
    for (y, x, h, w) in _windows(H, Wd):
        y0, x0 = max(0, y - W), max(0, x - W)
        y1, x1 = min(H, y + h + W), min(Wd, x + w + W)
        sub = orc.gpa(img[y0:y1, x0:x1].astype(np.float64), kind, W, k.weights_1d, sigma_r, N)
        worst = max(worst, float(np.max(np.abs(out[y:y + h, x:x + w] - sub[y - y0:y - y0 + h, x - x0:x - x0 + w]))))
    assert worst <= 1e-8, worst


@pytest.mark.parametrize("kind", ["box", "gaussian"])
@pytest.mark.parametrize("W", list(range(1, 33)))
def test_every_fast_half_width(kind, W):
    """Every half-width 1..32 has specialised kernels in both precisions (fb_tu_*_<group>.cu,
    fb_tu64_*_<group>.cu): each matches the oracle."""
    k = (make_spatial_kernel("box", half_width=W) if kind == "box"
         else make_spatial_kernel("gaussian", sigma_s=(W - 0.5) / 3.0))
    assert k.half_width == W
    rng = np.random.default_rng(100 + W)
    img = np.floor(rng.uniform(0.0, 256.0, (2 * W + 40, 2 * W + 70)))
    N = 25
    ref = orc.gpa(img, kind, W, k.weights_1d, 30.0, N)
    o32 = gpa_filter(img, k, 30.0, N, precision="f32")
    o64 = gpa_filter(img, k, 30.0, N, precision="f64")
    assert np.max(np.abs(o32 - ref)) <= F32_TOL
    assert np.max(np.abs(o64 - ref)) <= 1e-8


def test_graph_replay_of_small_repeated_calls():
    """Small device-resident calls repeat as CUDA-graph replays (fb_capi.cu): the same outputs
    as eager calls, new input contents honoured, kernels counted, per-kernel times -1."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(7)
    img = np.floor(rng.uniform(0.0, 256.0, (300, 280))).astype(np.float32)
    k = make_spatial_kernel("gaussian", sigma_s=3.0)
    src = torch.from_numpy(img).cuda()
    out = torch.empty_like(src)
    ref = orc.gpa(img.astype(np.float64), "gaussian", k.half_width, k.weights_1d, 40.0, 15)
    stats = []
    for _ in range(4):  # eager, capture, replay, replay
        n0 = _native.launch_count()
        st = _native.gpa(src, out, k, 40.0, 15, 128.0, 128.0, _native.FB_PREC_F32, 0)
        assert _native.launch_count() - n0 == 1  # the fused small-image kernel
        assert np.max(np.abs(out.cpu().numpy() - ref)) <= F32_TOL
        stats.append(st)
    assert stats[0]["k1_ms"] > 0 and stats[3]["k1_ms"] == -1.0 and stats[3]["kernel_ms"] > 0
    # same pointers, new contents: the replay reads the current input
    img2 = np.floor(rng.uniform(0.0, 256.0, img.shape)).astype(np.float32)
    src.copy_(torch.from_numpy(img2))
    _native.gpa(src, out, k, 40.0, 15, 128.0, 128.0, _native.FB_PREC_F32, 0)
    ref2 = orc.gpa(img2.astype(np.float64), "gaussian", k.half_width, k.weights_1d, 40.0, 15)
    assert np.max(np.abs(out.cpu().numpy() - ref2)) <= F32_TOL
    # an invalid sample still raises through a replayed graph (flags are part of the graph)
    src[5, 7] = 300.0
    from paper_1603_08109_b200 import RangeViolationError
    with pytest.raises(RangeViolationError, match=r"row=5, col=7"):
        _native.gpa(src, out, k, 40.0, 15, 128.0, 128.0, _native.FB_PREC_F32, 0)


def test_graph_replay_of_pinned_host_calls():
    """Small calls on page-locked host buffers replay as one CUDA graph too (H2D, kernels, D2H
    and the flag readback captured): same outputs, new input contents honoured, copy byte
    counts kept; pageable buffers stay eager and give the same result."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(9)
    img = np.floor(rng.uniform(0.0, 256.0, (300, 280)))
    k = make_spatial_kernel("box", half_width=5)
    src = torch.from_numpy(img).pin_memory().numpy()
    out = torch.empty(img.shape, dtype=torch.float64).pin_memory().numpy()
    ref = orc.gpa(img, "box", 5, k.weights_1d, 50.0, 10)
    stats = []
    for _ in range(5):  # eager (x2: the staging buffers appear in the key), capture, replay, replay
        st = _native.gpa(src, out, k, 50.0, 10, 128.0, 128.0, _native.FB_PREC_F32, 0)
        assert np.max(np.abs(out - ref)) <= F32_TOL
        assert st["h2d_bytes"] == src.nbytes and st["d2h_bytes"] == out.nbytes
        stats.append(st)
    assert stats[0]["k1_ms"] > 0 and stats[-1]["k1_ms"] == -1.0
    img2 = np.floor(rng.uniform(0.0, 256.0, img.shape))
    src[...] = img2
    _native.gpa(src, out, k, 50.0, 10, 128.0, 128.0, _native.FB_PREC_F32, 0)
    assert np.max(np.abs(out - orc.gpa(img2, "box", 5, k.weights_1d, 50.0, 10))) <= F32_TOL
    pageable_out = np.empty_like(out)
    for _ in range(3):
        st = _native.gpa(img2.copy(), pageable_out, k, 50.0, 10, 128.0, 128.0, _native.FB_PREC_F32, 0)
        assert st["k1_ms"] > 0  # never replayed
    assert np.array_equal(pageable_out, out)


@pytest.mark.parametrize("kind,param,sr,n,precision", [("box", 20, 25.0, 57, "f32"), ("gaussian", 8.0, 20.0, 40, "f32"),
                                                       ("box", 20, 25.0, 57, "f64"), ("gaussian", 5.0, 30.0, 42, "f64")])
def test_repeated_calls_are_bit_identical(kind, param, sr, n, precision):
    """Stage-ring races (a stage refilled while a lane still reads it) show up as run-to-run
    differences: repeated calls on the same device image must agree bit for bit."""
    torch = pytest.importorskip("torch")
    img = synth.config_image("c4", height=2048, width=4096)
    k = make_spatial_kernel(kind, **({"half_width": param} if kind == "box" else {"sigma_s": param}))
    d = torch.from_numpy(img).cuda()
    outs = [torch.empty(img.shape, dtype=torch.float64, device="cuda") for _ in range(6)]
    for o in outs:  # distinct output buffers: eager calls, no graph replay
        gpa_filter(d, k, sr, n, precision=precision, out=o)
    first = outs[0].cpu().numpy()
    for o in outs[1:]:
        assert np.array_equal(o.cpu().numpy(), first)


def test_fused_single_pass_prototype_matches(tmp_path):
    """The single-pass box kernel (fb_fused.cuh, selected by FBGPU_FUSED_BOX=1
    and read once per process, hence the subprocess) stays within the bar of the fp64 path."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, torch\n"
        "from paper_1603_08109_b200 import gpa_filter, make_spatial_kernel, synth\n"
        "img = synth.config_image('c4', height=2304, width=2048)\n"
        "k = make_spatial_kernel('box', half_width=20)\n"
        "d = torch.from_numpy(img).cuda()\n"
        "st = {}\n"
        "o32 = gpa_filter(d, k, 25.0, 57, precision='f32', stats=st).cpu().numpy()\n"
        "o64 = gpa_filter(d, k, 25.0, 57, precision='f64').cpu().numpy()\n"
        "print(float(np.max(np.abs(o32 - o64))), st['launches'])\n")
    env = dict(os.environ, FBGPU_FUSED_BOX="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    err, launches = r.stdout.split()
    assert float(err) <= 1e-3 and int(launches) == 1
