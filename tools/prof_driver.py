"""Minimal driver for ncu: filter one config image (device-resident) `--reps` times.

  ncu --set full -k regex:k2f -s 1 -c 1 -o gpurun_out/prof python tools/prof_driver.py --config c3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_08109_b200 import _native, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--rows", type=int, default=0, help="crop rows (0 = full image)")
ap.add_argument("--lib", default=None, help="alternative libfbgpu.so (A/B experiments)")
ap.add_argument("--e2e", action="store_true", help="time gpa_filter with pinned host in/out instead")
args = ap.parse_args()
if args.lib:
    _native.load_library(args.lib)
cfg = synth.CONFIGS[args.config]
img = synth.config_image(cfg)
if args.rows:
    img = np.ascontiguousarray(img[: args.rows])
k = synth.config_kernel(cfg)
N = synth.config_order(cfg)
if args.e2e:
    import time

    from paper_1603_08109_b200 import gpa_filter, gpa_filter_batch
    imgs = [img] + [synth.config_image(cfg, i) for i in range(1, cfg.batch)]
    pin = [torch.from_numpy(im).pin_memory().numpy() for im in imgs]
    pout = [torch.empty(im.shape, dtype=torch.float64).pin_memory().numpy() for im in imgs]
    best = 1e9
    for _ in range(args.reps + 1):
        t0 = time.perf_counter()
        if len(pin) > 1:
            gpa_filter_batch(pin, k, cfg.sigma_r, N, precision="f32", device=0, outs=pout)
        else:
            gpa_filter(pin[0], k, cfg.sigma_r, N, precision="f32", device=0, out=pout[0])
        best = min(best, time.perf_counter() - t0)
    px = sum(im.size for im in imgs)
    print(f"{args.lib or ''} {args.config} e2e {best * 1e3:.2f} ms = {px / best / 1e6:.0f} MP/s")
    sys.exit(0)
d = torch.from_numpy(img).cuda()
out = torch.empty(img.shape, dtype=torch.float32, device="cuda")
k1s, k2s = [], []
for _ in range(args.reps):
    st = _native.gpa(d, out, k, cfg.sigma_r, N, 128.0, 128.0, _native.FB_PREC_F32, 0)
    k1s.append(st["k1_ms"])
    k2s.append(st["k2_ms"])
torch.cuda.synchronize()
print(f"{args.lib or ''} {args.config} {img.shape} N={N} k1_ms={st['k1_ms']:.3f} k2_ms={st['k2_ms']:.3f} "
      f"median k1={np.median(k1s):.3f} k2={np.median(k2s):.3f} bands={st['bands']}")
