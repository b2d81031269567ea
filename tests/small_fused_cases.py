"""Run by tests/test_gpu_small.py in a subprocess with FBGPU_SMALL_FUSED=0 / 1 (the library reads
it once per process): filters c0 and c1 into c0.npy / c1.npy in the working directory, prints
the kernels each call launched, then runs the box cases of test_gpu_small.py under that setting."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_1603_08109_b200 import gpa_filter, synth  # noqa: E402

for name in ("c0", "c1"):
    cfg = synth.CONFIGS[name]
    st = {}
    o = gpa_filter(synth.config_image(cfg), synth.config_kernel(cfg), cfg.sigma_r, synth.config_order(cfg),
                   precision="f32", stats=st)
    np.save(f"{name}.npy", o)
    print(st["launches"])

import test_gpu_small as t  # noqa: E402

for case in ((300, 517, "box", 5, 50.0, 10, np.float32), (270, 261, "box", 1, 60.0, 8, np.uint8),
             (261, 300, "box", 20, 25.0, 57, np.float32), (257, 259, "box", 32, 60.0, 9, np.float32),
             (33, 2000, "box", 3, 40.0, 12, np.float32)):
    t.test_small_fused_matches_oracle(*case)
t.test_small_band_calls_are_bit_identical("box", 5, 50.0, 10)
t.test_small_band_calls_are_bit_identical("box", 20, 25.0, 30)
t.test_small_validation_names_the_first_offender()
print("ok")
