"""Host path of the fp32 precision for float64 outputs in host memory (csrc/fb_hostwiden.cuh): calls
of more than 16 MP send the float32 centred result over PCIe and host threads widen it into the
caller's float64 array.  The result must be the very bits of the device-resident call
(engine.py:27-80 returns float64; results do not depend on the decomposition)."""

import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1603_08109_b200 import gpa_filter, gpa_filter_batch, make_spatial_kernel

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _image(h, w, seed, dtype=np.float32):
    rng = np.random.default_rng(seed)
    img = rng.uniform(0.0, 255.0, (h, w))
    img[::97, ::89] = 255.0
    return img.astype(dtype)


def _device_call(img, k, sigma_r, N, **kw):
    import torch
    return gpa_filter(torch.from_numpy(img).cuda(), k, sigma_r, N, precision="f32", **kw).cpu().numpy()


@pytest.mark.parametrize("kind,param,sigma_r,N", [("box", 5, 50.0, 10), ("gaussian", 2.0, 40.0, 8), ("box", 20, 25.0, 57)])
def test_widened_host_output_is_bit_identical_to_device_call(kind, param, sigma_r, N):
    k = make_spatial_kernel("box", half_width=param) if kind == "box" else make_spatial_kernel("gaussian", sigma_s=param)
    img = _image(4200, 4100, 3)  # 17.2 MP: over the graph-replay limit, chunked, widened
    st = {}
    out = np.empty(img.shape, dtype=np.float64)  # pageable: the host threads write it directly
    gpa_filter(img, k, sigma_r, N, precision="f32", out=out, stats=st)
    assert st["d2h_bytes"] == img.size * 4 and st["h2d_bytes"] == img.size * 4
    ref = _device_call(img, k, sigma_r, N)
    assert np.array_equal(out, ref)
    # the fp32 path's centred results are fp32 values (default range: t_c = 128)
    c = ref - 128.0
    assert np.array_equal(c, c.astype(np.float32).astype(np.float64))


def test_float64_input_keeps_the_float64_transfer():
    k = make_spatial_kernel("box", half_width=3)
    img = _image(4200, 4100, 4, np.float64)
    st = {}
    out = gpa_filter(img, k, 30.0, 6, precision="f32", stats=st)
    assert st["d2h_bytes"] == img.size * 8
    assert np.array_equal(out, _device_call(img, k, 30.0, 6))


def test_widened_batch_matches_single_calls():
    k = make_spatial_kernel("gaussian", sigma_s=1.5)
    imgs = [_image(1500, 1400, 10 + i) for i in range(9)]  # 18.9 MP in all: widened per image
    st = {}
    outs = gpa_filter_batch(imgs, k, 35.0, 7, precision="f32", stats=st)
    assert st["d2h_bytes"] == sum(im.size for im in imgs) * 4
    for im, o in zip(imgs, outs):
        assert o.dtype == np.float64
        assert np.array_equal(o, _device_call(im, k, 35.0, 7))


def test_degenerate_pixels_repeat_the_call_with_float64_rows():
    """A pixel under the Q floor returns the input sample (engine.py:68): the call then runs again
    without the float32 transfer, so the sample comes back exactly."""
    k = make_spatial_kernel("box", half_width=1)
    img = np.zeros((4200, 4100), dtype=np.float32)  # sigma_r = 10: Q underflows away from the bright pixels
    img[::50, ::50] = 255.0
    st = {}
    out = gpa_filter(img, k, 10.0, 1, allow_small_sigma=True, precision="f32", stats=st)
    assert st["degenerate_pixels"] > 0
    assert st["d2h_bytes"] == img.size * 8
    assert np.array_equal(out, _device_call(img, k, 10.0, 1, allow_small_sigma=True))


def test_host_threads_zero_disables_the_float32_transfer():
    code = (
        "import numpy as np\n"
        "from paper_1603_08109_b200 import gpa_filter, make_spatial_kernel\n"
        "rng = np.random.default_rng(3)\n"
        "img = rng.uniform(0.0, 255.0, (4200, 4100)).astype(np.float32)\n"
        "st = {}\n"
        "out = gpa_filter(img, make_spatial_kernel('box', half_width=5), 50.0, 10, precision='f32', stats=st)\n"
        "np.save('o.npy', out)\n"
        "print(st['d2h_bytes'])\n")
    import tempfile
    outs = {}
    # (threads, staging limit in MB) -> bytes per pixel over PCIe: no threads or no room for the
    # pinned staging area mean float64 rows
    for key, env_add, bpp in (("off", {"FBGPU_HOST_THREADS": "0"}, 8), ("on", {"FBGPU_HOST_THREADS": "3"}, 4),
                              ("no_room", {"FBGPU_HOST_THREADS": "3", "FBGPU_WIDEN_MAX_MB": "1"}, 8)):
        with tempfile.TemporaryDirectory() as tmp:
            env = dict(os.environ, PYTHONPATH=ROOT, **env_add)
            r = subprocess.run([sys.executable, "-c", code], env=env, cwd=tmp, capture_output=True, text=True, timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            assert int(r.stdout.split()[-1]) == 4200 * 4100 * bpp, key
            outs[key] = np.load(os.path.join(tmp, "o.npy"))
    assert np.array_equal(outs["off"], outs["on"])
    assert np.array_equal(outs["off"], outs["no_room"])
