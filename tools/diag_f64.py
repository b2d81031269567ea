"""fp32 vs fp64 kernel times on the c2 image and a 4096-row c4 band (device-resident).

  python tools/diag_f64.py [--lib abtest/NAME.so]
"""
import argparse
import os
import sys

os.environ.setdefault("FBGPU_NO_GRAPHS", "1")  # per-kernel times need eager calls
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1603_08109_b200 import _native, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
args = ap.parse_args()
if args.lib:
    _native.load_library(args.lib)
for name in ("c2", "c4"):
    cfg = synth.CONFIGS[name]
    img = synth.config_image(cfg, height=4096 if name == "c4" else None)
    k = synth.config_kernel(cfg)
    N = synth.config_order(cfg)
    d = torch.from_numpy(img).cuda()
    out = torch.empty(img.shape, dtype=torch.float64, device="cuda")
    for prec, tag in ((_native.FB_PREC_F32, "f32"), (_native.FB_PREC_F64, "f64")):
        _native.gpa(d, out, k, cfg.sigma_r, N, 128.0, 128.0, prec, 0)
        st = _native.gpa(d, out, k, cfg.sigma_r, N, 128.0, 128.0, prec, 0)
        ms = st["k1_ms"] + st["k2_ms"]
        print(args.lib or "", name, tuple(img.shape), tag,
              f"k1 {st['k1_ms']:.2f} k2 {st['k2_ms']:.2f} ms -> {img.size / ms / 1e3:.0f} MP/s")
