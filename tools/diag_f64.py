import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1603_08109_b200 import _native, synth
for name in ("c2", "c4"):
    cfg = synth.CONFIGS[name]
    img = synth.config_image(cfg, height=4096 if name == "c4" else None)
    k = synth.config_kernel(cfg); N = synth.config_order(cfg)
    d = torch.from_numpy(img).cuda(); out = torch.empty(img.shape, dtype=torch.float64, device="cuda")
    for prec, tag in ((_native.FB_PREC_F32, "f32"), (_native.FB_PREC_F64, "f64")):
        st = _native.gpa(d, out, k, cfg.sigma_r, N, 128.0, 128.0, prec, 0)
        st = _native.gpa(d, out, k, cfg.sigma_r, N, 128.0, 128.0, prec, 0)
        print(name, img.shape, tag, f"k1 {st['k1_ms']:.2f} k2 {st['k2_ms']:.2f} ms -> {img.size/(st['k1_ms']+st['k2_ms'])/1e3:.0f} MP/s")
