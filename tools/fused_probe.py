"""The single-pass box kernel (fb_fused.cuh) against the two-kernel path: accuracy vs the fp64
path and time per c4 band.  Run once with FBGPU_FUSED_BOX=1 and once without (the switch is read
once per process):

  FBGPU_FUSED_BOX=1 python tools/fused_probe.py ; python tools/fused_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_08109_b200 import _native, gpa_filter, make_spatial_kernel, synth  # noqa: E402

tag = "fused" if os.environ.get("FBGPU_FUSED_BOX", "0") not in ("", "0") else "two-kernel"
k = make_spatial_kernel("box", half_width=20)
# accuracy on a c4-recipe image (walker territory), fp32 output vs the fp64 path
img = synth.config_image("c4", height=2304, width=2048)
d = torch.from_numpy(img).cuda()
o32 = gpa_filter(d, k, 25.0, 57, precision="f32").cpu().numpy()
o64 = gpa_filter(d, k, 25.0, 57, precision="f64").cpu().numpy()
err = float(np.max(np.abs(o32 - o64)))
# one c4 band: 4096 x 16384, N = 57
band = torch.from_numpy(synth.config_image("c4")[:4096].copy()).cuda()
out = torch.empty(band.shape, dtype=torch.float32, device="cuda")
ms = []
for _ in range(6):
    st = _native.gpa(band, out, k, 25.0, 57, 128.0, 128.0, _native.FB_PREC_F32, 0)
    ms.append(st["kernel_ms"])
print(f"{tag}: max|f32 - f64| = {err:.3e} on 2304x2048; c4 band kernel time median {np.median(ms[1:]):.3f} ms "
      f"(k1 {st['k1_ms']:.3f}, k2 {st['k2_ms']:.3f}); {st['launches']} launches", flush=True)
