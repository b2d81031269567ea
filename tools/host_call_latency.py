"""Wall time per gpa_filter call with pinned host buffers for the small configs (graph-replayed calls).
  python tools/host_call_latency.py [alternative libfbgpu.so]"""
import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1603_08109_b200 import _native, gpa_filter, synth
if len(sys.argv) > 1:
    _native.load_library(sys.argv[1])
for name in ("c0", "c1"):
    cfg = synth.CONFIGS[name]; N = synth.config_order(cfg); k = synth.config_kernel(cfg)
    img = torch.from_numpy(synth.config_image(cfg)).pin_memory().numpy()
    out = torch.empty(img.shape, dtype=torch.float64).pin_memory().numpy()
    st = {}
    for i in range(5): gpa_filter(img, k, cfg.sigma_r, N, precision="f32", out=out, stats=st)
    t0 = time.perf_counter()
    for i in range(300): gpa_filter(img, k, cfg.sigma_r, N, precision="f32", out=out, stats=st)
    dt = (time.perf_counter() - t0) / 300 * 1e3
    print(name, f"host call {dt:.3f} ms  k1_ms {st['k1_ms']} device_ms {st['device_ms']:.3f} launches {st['launches']}")
    t0 = time.perf_counter()
    for i in range(300): gpa_filter(img, k, cfg.sigma_r, N, precision="f32", out=out)
    print(name, f"  without stats {(time.perf_counter() - t0) / 300 * 1e3:.3f} ms")
