"""Precision study: max |fp32 path - fp64 path| over seeded images for a grid of (kernel, sigma_r).

  FBGPU_HORNER=32 python tools/precision_sweep.py --tag h32
  FBGPU_HORNER=64 python tools/precision_sweep.py --tag h64
Writes profiles/precision_<tag>.json; used to set the Horner-precision policy.
"""
import argparse, json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1603_08109_b200 import gpa_filter, make_spatial_kernel, synth, epsilon_from_delta, estimate_order

ap = argparse.ArgumentParser()
ap.add_argument("--tag", required=True)
ap.add_argument("--size", type=int, default=2048)
ap.add_argument("--images", type=int, default=2)
args = ap.parse_args()
kernels = [("box", 5), ("box", 20), ("gaussian", 3.0), ("gaussian", 5.0), ("gaussian", 8.0)]
sigmas = [16.0, 20.0, 25.0, 30.0, 40.0, 50.0]
res = []
for kind, p in kernels:
    k = make_spatial_kernel(kind, half_width=p) if kind == "box" else make_spatial_kernel(kind, sigma_s=p)
    for sr in sigmas:
        N = estimate_order(sr, epsilon_from_delta(1.0, k.w0, 128.0), 128.0).N0
        worst = 0.0
        for i in range(args.images):
            cfg = "c4" if i % 2 == 0 else "c2"
            img = synth.config_image(cfg, i, height=args.size, width=args.size)
            o32 = gpa_filter(img, k, sr, N, precision="f32")
            o64 = gpa_filter(img, k, sr, N, precision="f64")
            worst = max(worst, float(np.max(np.abs(o32 - o64))))
        res.append({"kind": kind, "param": p, "sigma_r": sr, "N": N, "max_abs": worst})
        print(json.dumps(res[-1]), flush=True)
with open(os.path.join(ROOT, "profiles", f"precision_{args.tag}.json"), "w") as fh:
    json.dump({"horner": os.environ.get("FBGPU_HORNER", "auto"), "size": args.size, "images": args.images,
               "results": res}, fh, indent=1)
