"""Per-call latency of small filters: wall time of one synchronous call vs the device time it
spans (ev_start..ev_end inside the C ABI) and the kernel time.

  python tools/diag_latency.py [--config c0]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_08109_b200 import _native, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c0")
ap.add_argument("--calls", type=int, default=200)
args = ap.parse_args()
cfg = synth.CONFIGS[args.config]
img = synth.config_image(cfg)
k = synth.config_kernel(cfg)
N = synth.config_order(cfg)
d = torch.from_numpy(img).cuda()
out = torch.empty(img.shape, dtype=torch.float32, device="cuda")
for _ in range(10):
    _native.gpa(d, out, k, cfg.sigma_r, N, 128.0, 128.0, _native.FB_PREC_F32, 0)
torch.cuda.synchronize()
walls, devs, kers = [], [], []
for _ in range(args.calls):
    t0 = time.perf_counter()
    st = _native.gpa(d, out, k, cfg.sigma_r, N, 128.0, 128.0, _native.FB_PREC_F32, 0)
    walls.append(time.perf_counter() - t0)
    devs.append(st["device_ms"])
    kers.append(st["kernel_ms"])  # graph replays report only the total (k1_ms = k2_ms = -1)
med = lambda v: float(np.median(v))  # noqa: E731
print(f"{args.config} {img.shape}: wall {med(walls) * 1e3:.3f} ms, device span {med(devs):.3f} ms, "
      f"kernels + flag copies {med(kers):.3f} ms")
