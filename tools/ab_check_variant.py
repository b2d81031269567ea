"""A/B numerics: `tools/ab_check_variant.py` saves the in-tree library's f32/f64 outputs, then
`tools/ab_check_variant.py abtest/X.so` compares the variant's f32 output with them."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_08109_b200 import _native, synth  # noqa: E402


def run(img, k, sr, N, prec):
    d = torch.from_numpy(img).cuda()
    out = torch.empty(img.shape, dtype=torch.float64, device="cuda")
    _native.gpa(d, out, k, sr, N, 128.0, 128.0, prec, 0)
    torch.cuda.synchronize()
    return out.cpu().numpy()


cases = []
for c, rows in (("c1", 0), ("c4", 1024)):
    cfg = synth.CONFIGS[c]
    img = synth.config_image(cfg)
    if rows:
        img = np.ascontiguousarray(img[:rows, :4096])
    cases.append((c, img, synth.config_kernel(cfg), cfg.sigma_r, synth.config_order(cfg)))
# isolated outliers (tiny Q at the outlier pixels)
cfg = synth.CONFIGS["c4"]
img = np.full((256, 512), 5.0, np.float32)
img[::37, ::41] = 250.0
cases.append(("outliers", img, synth.config_kernel(cfg), 10.0, synth.config_order(cfg)))

lib = sys.argv[1] if len(sys.argv) > 1 else None
if lib:
    _native.load_library(lib)
ref_path = "/tmp/ab_base.npz"
out = {}
for name, img, k, sr, N in cases:
    out[name] = run(img, k, sr, N, _native.FB_PREC_F32)
    if lib is None:
        out[name + "_f64"] = run(img, k, sr, N, _native.FB_PREC_F64)
if lib is None:
    os.makedirs(os.path.dirname(ref_path), exist_ok=True)
    np.savez(ref_path, **out)
    sys.exit(0)
ref = np.load(ref_path)
for name, *_ in cases:
    var, base, f64 = out[name], ref[name], ref[name + "_f64"]
    print(f"{name}: |var-base| {np.abs(var - base).max():.3e}  |base-f64| {np.abs(base - f64).max():.3e}  "
          f"|var-f64| {np.abs(var - f64).max():.3e}  finite {np.isfinite(var).all()}")
