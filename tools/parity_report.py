"""Full-size parity of the fp32 path: max |delta| per config on the WHOLE image.

The fp64 instantiation of the same kernels is the full-size reference here: it
matches the reference package's float64 outputs to <= 1e-9 on every golden case
(tests/test_gpu_parity.py), and the numpy oracle cannot run 268 MP in reasonable
time.  A few windows per config are additionally checked against the oracle
itself (interior exactness of the local filter).  Writes profiles/parity_<tag>.json.

  python tools/parity_report.py --tag r01 [--configs c0,c1,c2,c3,c4] [--c3-images 4]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import gpa_oracle as orc  # noqa: E402  (checker only)
from paper_1603_08109_b200 import bilateral_exact, gpa_filter, synth  # noqa: E402


def psnr(mse):
    """20 log10(255) - mse_db (analysis.py:41-46)."""
    import math
    return math.inf if mse == 0 else 20 * math.log10(255.0) - 10 * math.log10(mse)


def window_errs(img, out, k, sigma_r, N, windows):
    W = k.half_width
    H, Wd = img.shape
    worst = 0.0
    for (y, x, h, w) in windows:
        y0, x0 = max(0, y - W), max(0, x - W)
        y1, x1 = min(H, y + h + W), min(Wd, x + w + W)
        sub = orc.gpa(img[y0:y1, x0:x1], k.kind, W, k.weights_1d, sigma_r, N)
        ref = sub[y - y0:y - y0 + h, x - x0:x - x0 + w]
        worst = max(worst, float(np.max(np.abs(out[y:y + h, x:x + w] - ref))))
    return worst


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--configs", default="c0,c1,c2,c3,c4")
    ap.add_argument("--c3-images", type=int, default=4)
    args = ap.parse_args()
    report = {"tag": args.tag, "bar": 1e-3, "configs": {}}
    for name in args.configs.split(","):
        cfg = synth.CONFIGS[name]
        k = synth.config_kernel(cfg)
        N = synth.config_order(cfg)
        n_img = min(cfg.batch, args.c3_images) if cfg.batch > 1 else 1
        worst, worst_at, q9999, over1e4, npx = 0.0, None, [], 0, 0
        approx = {"ours_linf": 0.0, "ref_linf": 0.0, "ours_se": 0.0, "ref_se": 0.0}
        t0 = time.time()
        for i in range(n_img):
            img = synth.config_image(cfg, i)
            o32 = gpa_filter(img, k, cfg.sigma_r, N, precision="f32")
            o64 = gpa_filter(img, k, cfg.sigma_r, N, precision="f64")
            bf = bilateral_exact(img, k, cfg.sigma_r)  # GPU fp64 brute force
            e32, e64 = np.abs(o32 - bf), np.abs(o64 - bf)
            approx["ours_linf"] = max(approx["ours_linf"], float(e32.max()))
            approx["ref_linf"] = max(approx["ref_linf"], float(e64.max()))
            approx["ours_se"] += float(np.sum(e32 * e32))
            approx["ref_se"] += float(np.sum(e64 * e64))
            del bf, e32, e64
            d = np.abs(o32 - o64)
            j = np.unravel_index(int(np.argmax(d)), d.shape)
            if d[j] > worst:
                worst, worst_at = float(d[j]), [i, int(j[0]), int(j[1]), float(img[j])]
            q9999.append(float(np.quantile(d, 0.9999)))
            over1e4 += int((d > 1e-4).sum())
            npx += d.size
            H, Wd = img.shape
            wins = [(0, 0, 40, 40), (H - 40, Wd - 40, 40, 40), (H // 2, Wd // 3, 48, 48)]
            if worst_at and worst_at[0] == i:
                y, x = worst_at[1], worst_at[2]
                wins.append((max(0, y - 8), max(0, x - 8), min(16, H - max(0, y - 8)), min(16, Wd - max(0, x - 8))))
            w32 = window_errs(img, o32, k, cfg.sigma_r, N, wins)
            w64 = window_errs(img, o64, k, cfg.sigma_r, N, wins)
            del o32, o64, d
        report["configs"][name] = {
            "images": n_img, "pixels_compared": npx, "order_N": N, "kind": cfg.kind,
            "half_width": k.half_width, "sigma_r": cfg.sigma_r,
            "max_abs_f32_vs_f64": worst, "worst_pixel": worst_at,
            "p99.99_abs": max(q9999), "pixels_over_1e-4": over1e4,
            "windows_max_abs_f32_vs_oracle": w32, "windows_max_abs_f64_vs_oracle": w64,
            "seconds": round(time.time() - t0, 1),
            # approximation error vs the exact bilateral filter (GPU fp64 brute force): ours (fp32
            # path) and the reference-equivalent fp64 path (= the reference's gpa_filter to 1e-13)
            "approx_linf_ours": approx["ours_linf"], "approx_linf_reference": approx["ref_linf"],
            "approx_psnr_ours": psnr(approx["ours_se"] / npx), "approx_psnr_reference": psnr(approx["ref_se"] / npx),
        }
        print(name, json.dumps(report["configs"][name]), flush=True)
    out = os.path.join(ROOT, "profiles", f"parity_{args.tag}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        json.dump(report, fh, indent=1)


if __name__ == "__main__":
    main()
