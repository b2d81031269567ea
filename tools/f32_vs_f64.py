"""max |fp32 path - fp64 path| on a crop generated with a config's recipe (device-resident calls)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_08109_b200 import gpa_filter, synth  # noqa: E402

for name, h, w in (("c4", 2304, 2048), ("c4", 4096, 4096), ("c1", 1024, 1024), ("c2", 2048, 2048), ("c3", 2048, 2048)):
    cfg = synth.CONFIGS[name]
    img = synth.config_image(cfg, height=h, width=w)
    k = synth.config_kernel(cfg)
    N = synth.config_order(cfg)
    o32 = gpa_filter(img, k, cfg.sigma_r, N, precision="f32")
    o64 = gpa_filter(img, k, cfg.sigma_r, N, precision="f64")
    d = np.abs(o32 - o64)
    print(f"{name} {h}x{w} N={N}: max|f32-f64| {d.max():.3e}  mean {d.mean():.3e}  p99.9 {np.quantile(d, 0.999):.3e}", flush=True)
