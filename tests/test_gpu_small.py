"""GPU parity of the fused small-image kernel (csrc/fb_small.cuh): images of fewer than 2 Mi padded
samples on the fp32 path run gpa_filter (engine.py:27-80) in one kernel per 32 x 32 tile, the
channels generated, filtered (conv.py:30-64) and accumulated without leaving the SM.  It is the
default for Gaussian windows; box windows keep kernel 1 + kernel 2 unless FBGPU_SMALL_FUSED=1
(read once per process: the box cases of this module run again under it in a subprocess,
tests/small_fused_cases.py).

Whole images are compared with the oracle (pinned to the reference) and with the fp64 path; band
calls, batches and the two-kernel path must agree with the whole-image call.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import gpa_oracle as orc
from paper_1603_08109_b200 import (ParameterError, RangeViolationError, _native, gpa_filter, make_spatial_kernel,
                                   synth)

pytestmark = pytest.mark.gpu

F32_TOL = 1e-3


def _launches(kind):
    """Kernels per band: the fused kernel for Gaussian windows (and for box windows when forced)."""
    return 1 if kind == "gaussian" or os.environ.get("FBGPU_SMALL_FUSED") == "1" else 2


def _kernel(kind, param):
    return make_spatial_kernel("box", half_width=param) if kind == "box" else make_spatial_kernel("gaussian", sigma_s=param)


@pytest.mark.parametrize("h,w,kind,param,sigma_r,N,dtype", [
    (300, 280, "gaussian", 3.0, 40.0, 15, np.float64),   # c0's filter
    (300, 517, "box", 5, 50.0, 10, np.float32),          # c1's filter, ragged right edge
    (270, 261, "box", 1, 60.0, 8, np.uint8),             # narrowest window, 8-bit input
    (290, 300, "gaussian", 0.5, 30.0, 20, np.float32),   # W = 2
    (261, 300, "box", 20, 25.0, 57, np.float32),         # c4's filter on a small image
    (300, 290, "gaussian", 5.0, 30.0, 42, np.float32),   # c2's filter (W = 15)
    (280, 260, "gaussian", 8.0, 20.0, 76, np.float32),   # c3's filter (W = 24, 16-row vertical groups)
    (257, 259, "box", 32, 60.0, 9, np.float32),          # widest fast window
    (33, 2000, "box", 3, 40.0, 12, np.float32),          # one tile row and a bit, wide
    (2000, 31, "gaussian", 2.0, 45.0, 14, np.float32),   # narrower than a tile, tall
])
def test_small_fused_matches_oracle(h, w, kind, param, sigma_r, N, dtype):
    rng = np.random.default_rng(h * 7 + w)
    img = np.floor(rng.uniform(0.0, 256.0, (h, w))).astype(dtype)
    k = _kernel(kind, param)
    st = {}
    o32 = gpa_filter(img, k, sigma_r, N, precision="f32", stats=st)
    assert st["launches"] == _launches(kind) and st["bands"] == 1
    ref = orc.gpa(img.astype(np.float64), kind, k.half_width, k.weights_1d, sigma_r, N)
    assert np.max(np.abs(o32 - ref)) <= F32_TOL
    o64 = gpa_filter(img, k, sigma_r, N, precision="f64")
    assert np.max(np.abs(o64 - ref)) <= 1e-8


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_small_configs_every_pixel(name):
    """Every pixel of c0 (512^2 Gaussian) and c1 (1024^2 box) against the oracle."""
    cfg = synth.CONFIGS[name]
    img = synth.config_image(cfg)
    k = synth.config_kernel(cfg)
    N = synth.config_order(cfg)
    st = {}
    out = gpa_filter(img, k, cfg.sigma_r, N, precision="f32", stats=st)
    assert st["launches"] == _launches(cfg.kind)
    ref = orc.gpa(img.astype(np.float64), cfg.kind, k.half_width, k.weights_1d, cfg.sigma_r, N)
    assert np.max(np.abs(out - ref)) <= 1e-4


@pytest.mark.parametrize("kind,param,sigma_r,N", [("box", 5, 50.0, 10), ("box", 20, 25.0, 30), ("gaussian", 3.0, 40.0, 15)])
def test_small_band_calls_are_bit_identical(kind, param, sigma_r, N):
    """Row bands of a small image (fb_gpa_filter_band, halo rows in separate buffers) give the bits
    of the whole-image call: box tiles and their running-sum groups are anchored to image rows
    (SPEC.md:322)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    H, Wd = 700, 333
    img = np.floor(rng.uniform(0.0, 256.0, (H, Wd))).astype(np.float32)
    k = _kernel(kind, param)
    W = k.half_width
    full = gpa_filter(torch.from_numpy(img).cuda(), k, sigma_r, N, precision="f32").cpu().numpy()
    # bands on the 32-row tile grid need W halo rows; a band off the grid re-walks the rows of the
    # tile above its first row (lead), so it carries W + r0 % 32 rows above
    for r0, r1, top in ((0, 256, 0), (256, 512, W), (512, H, W), (100, 431, W + 100 % 32), (37, 38, W + 37 % 32)):
        top = min(top, r0)
        band = torch.from_numpy(np.ascontiguousarray(img[r0:r1])).cuda()
        above = torch.from_numpy(np.ascontiguousarray(img[r0 - top:r0])).cuda() if top else None
        nb = min(W, H - r1)
        below = torch.from_numpy(np.ascontiguousarray(img[r1:r1 + nb])).cuda() if nb else None
        out = torch.empty((r1 - r0, Wd), dtype=torch.float64, device="cuda")
        st = _native.gpa_band(band, out, k, sigma_r, N, 128.0, 128.0, _native.FB_PREC_F32, r0, H, above, below, 0)
        assert st["launches"] == _launches(kind)
        assert np.array_equal(out.cpu().numpy(), full[r0:r1]), (r0, r1)


def test_small_output_dtypes_and_strides():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(11)
    img = np.floor(rng.uniform(0.0, 256.0, (301, 263))).astype(np.float32)
    k = make_spatial_kernel("gaussian", sigma_s=2.0)
    o64 = gpa_filter(img, k, 40.0, 15, precision="f32")
    o32 = gpa_filter(img, k, 40.0, 15, precision="f32", out_dtype=np.float32)
    o8 = gpa_filter(img, k, 40.0, 15, precision="f32", out_dtype=np.uint8)
    assert o64.dtype == np.float64 and np.array_equal(o32, o64.astype(np.float32))
    assert np.array_equal(o8, orc.quantize_u8(o64))
    # a strided device view in, a strided device view out
    big = torch.zeros((301, 400), dtype=torch.float32, device="cuda")
    big[:, 50:313] = torch.from_numpy(img).cuda()
    outbig = torch.full((301, 300), -1.0, dtype=torch.float64, device="cuda")
    _native.gpa(big[:, 50:313], outbig[:, 20:283], k, 40.0, 15, 128.0, 128.0, _native.FB_PREC_F32, 0)
    assert np.array_equal(outbig[:, 20:283].cpu().numpy(), o64)
    assert float(outbig[:, :20].max()) == -1.0 and float(outbig[:, 283:].max()) == -1.0


def test_small_validation_names_the_first_offender():
    rng = np.random.default_rng(2)
    img = np.floor(rng.uniform(0.0, 256.0, (300, 270))).astype(np.float32)
    k = make_spatial_kernel("box", half_width=4)
    bad = img.copy()
    bad[200, 33] = 400.0
    bad[77, 260] = 300.0
    bad[77, 269] = -1.0
    with pytest.raises(RangeViolationError, match=r"sample 300.0 at pixel \(row=77, col=260\)"):
        gpa_filter(bad, k, 40.0, 12, precision="f32")
    bad[150, 0] = np.inf
    with pytest.raises(ParameterError, match="non-finite"):
        gpa_filter(bad, k, 40.0, 12, precision="f32")


def test_small_fused_agrees_with_two_kernels():
    """FBGPU_SMALL_FUSED (read once per process) = 1 fuses box windows too, = 0 keeps kernel 1 +
    kernel 2 everywhere: the same filter to fp32 rounding of the planes on c0 and c1, and the
    box cases of this module hold on the fused kernel (tests/small_fused_cases.py)."""
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = os.path.join(root, "tests", "small_fused_cases.py")
    outs = {}
    for flag, launches in (("1", "1"), ("0", "2")):
        with tempfile.TemporaryDirectory() as tmp:
            env = dict(os.environ, FBGPU_SMALL_FUSED=flag, PYTHONPATH=root)
            r = subprocess.run([sys.executable, script], env=env, cwd=tmp, capture_output=True, text=True,
                               timeout=900)
            assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])
            assert r.stdout.split()[:2] == [launches, launches]
            outs[flag] = [np.load(os.path.join(tmp, f"{n}.npy")) for n in ("c0", "c1")]
    for a, b in zip(outs["1"], outs["0"]):
        assert np.max(np.abs(a - b)) <= 1e-4
