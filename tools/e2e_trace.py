"""Wall time of gpa_filter(pinned float32 in, out= pinned float64) per call for one config.
FBGPU_HOST_THREADS selects the host widening (0: float64 over PCIe), FBGPU_WIDEN_TRACE=1 prints
the worker timeline of each call."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_08109_b200 import gpa_filter, synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
N = synth.config_order(cfg)
k = synth.config_kernel(cfg)
img = torch.from_numpy(synth.config_image(cfg)).pin_memory().numpy()
out = torch.empty(img.shape, dtype=torch.float64).pin_memory().numpy()
ts = []
for i in range(6):
    st = {}
    t0 = time.perf_counter()
    gpa_filter(img, k, cfg.sigma_r, N, precision="f32", out=out, stats=st)
    ts.append((time.perf_counter() - t0) * 1e3)
    print(f"call {i}: wall {ts[-1]:.2f} ms  device {st['device_ms']:.2f} ms  kernels {st.get('k1_ms', 0) + st.get('k2_ms', 0):.2f} ms "
          f"d2h {st['d2h_bytes'] / 2**20:.0f} MiB", flush=True)
px = img.size / 1e6
print(f"{cfg.name} threads={os.environ.get('FBGPU_HOST_THREADS')} best {min(ts):.2f} ms = {px / min(ts) * 1e3:.0f} MP/s")
