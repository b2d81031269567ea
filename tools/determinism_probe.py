"""Run-to-run determinism of the filter on one device image (a stage-ring race shows up as
differing outputs).  python tools/determinism_probe.py [--lib abtest/NAME.so] [--reps 8]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_08109_b200 import _native, gpa_filter, make_spatial_kernel, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--reps", type=int, default=8)
args = ap.parse_args()
if args.lib:
    _native.load_library(args.lib)
img = synth.config_image("c4", height=2048, width=4096)
d = torch.from_numpy(img).cuda()
for kind, prm, sr, n, prec in (("box", 20, 25.0, 57, "f32"), ("gaussian", 8.0, 20.0, 40, "f32"), ("box", 20, 25.0, 57, "f64")):
    k = make_spatial_kernel(kind, **({"half_width": prm} if kind == "box" else {"sigma_s": prm}))
    outs = [torch.empty(img.shape, dtype=torch.float64, device="cuda") for _ in range(args.reps)]
    for o in outs:
        gpa_filter(d, k, sr, n, precision=prec, out=o)
    ref = outs[0].cpu().numpy()
    diffs = [float(np.max(np.abs(o.cpu().numpy() - ref))) for o in outs[1:]]
    print(args.lib or "in-tree", kind, prec, "max run-to-run diff", max(diffs), "identical runs", sum(x == 0 for x in diffs))
