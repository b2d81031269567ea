"""Small-image fused kernel (fb_small.cuh) vs the fp64 path on the full c0 / c1 images and on odd
shapes, plus its eager kernel time next to kernel 1 + kernel 2 (FBGPU_SMALL_FUSED=0).

  python tools/small_check.py            # parity + this process's kernel times
  FBGPU_SMALL_FUSED=0 python tools/small_check.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FBGPU_NO_GRAPHS", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_08109_b200 import _native, gpa_filter, make_spatial_kernel, synth  # noqa: E402

mode = "k1+k2" if os.environ.get("FBGPU_SMALL_FUSED") == "0" else "fused"
for name in ("c0", "c1"):
    cfg = synth.CONFIGS[name]
    img = synth.config_image(cfg)
    k = synth.config_kernel(cfg)
    N = synth.config_order(cfg)
    d = torch.from_numpy(img).cuda()
    o32 = gpa_filter(d, k, cfg.sigma_r, N, precision="f32").cpu().numpy()
    o64 = gpa_filter(d, k, cfg.sigma_r, N, precision="f64").cpu().numpy()
    out = torch.empty(img.shape, dtype=torch.float32, device="cuda")
    ks = []
    for _ in range(30):
        st = _native.gpa(d, out, k, cfg.sigma_r, N, 128.0, 128.0, _native.FB_PREC_F32, 0)
        ks.append((st["k1_ms"], st["k2_ms"], st["device_ms"]))
    k1, k2, dev = np.median(np.array(ks), axis=0)
    print(f"{mode} {name} {img.shape} N={N}: max|f32-f64| {np.max(np.abs(o32 - o64)):.3e}  "
          f"k1 {k1 * 1e3:.1f} us  k2-k1end {k2 * 1e3:.1f} us  device span {dev * 1e3:.1f} us")

rng = np.random.default_rng(5)
worst = 0.0
for (h, w, kind, W, sr, N) in ((300, 517, "box", 3, 30.0, 12), (261, 300, "gaussian", 2, 40.0, 9),
                               (700, 333, "box", 20, 25.0, 30), (513, 600, "gaussian", 11, 20.0, 40),
                               (400, 290, "box", 32, 60.0, 8), (290, 400, "gaussian", 32, 50.0, 11),
                               (1000, 1000, "gaussian", 24, 20.0, 76)):
    img = np.floor(rng.uniform(0, 256, (h, w))).astype(np.float32)
    k = make_spatial_kernel(kind, half_width=W) if kind == "box" else make_spatial_kernel(kind, sigma_s=W / 3.0)
    d = torch.from_numpy(img).cuda()
    e = float(np.max(np.abs(gpa_filter(d, k, sr, N, precision="f32").cpu().numpy()
                            - gpa_filter(d, k, sr, N, precision="f64").cpu().numpy())))
    worst = max(worst, e)
    print(f"{mode} {h}x{w} {kind} W={k.half_width} sr={sr} N={N}: max|f32-f64| {e:.3e}")
print("worst", worst)
assert worst <= 1e-3
