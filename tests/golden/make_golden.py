"""Generate the golden fixtures from the REFERENCE package itself.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It writes `tests/golden/reference_golden.npz` (inputs + the reference's float64
outputs) and `tests/golden/reference_scalars.json` (orders, epsilons, errors).
The GPU box never runs this script (`/root/reference` does not exist there);
tests only read the committed fixtures.  Inputs of the config cases are crops
of the seeded synthetic config images (`paper_1603_08109_b200/synth.py`).
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
if os.path.isdir("/root/reference/pkg/src"):
    sys.path.insert(0, "/root/reference/pkg/src")

import fastbilateral as fb  # noqa: E402  (the reference)

from paper_1603_08109_b200 import synth  # noqa: E402

CROP = (72, 88)  # non-square on purpose


def ref_kernel(cfg):
    if cfg.kind == "box":
        return fb.make_spatial_kernel("box", half_width=cfg.half_width)
    return fb.make_spatial_kernel("gaussian", sigma_s=cfg.sigma_s)


def main():
    arrays: dict[str, np.ndarray] = {}
    scalars: dict = {"reference_version": fb.__version__, "cases": {}}

    # ---- config crops -------------------------------------------------------
    for name, cfg in synth.CONFIGS.items():
        full = synth.config_image(cfg)
        h, w = full.shape
        y0, x0 = h // 2 - CROP[0] // 2, w // 3
        crop = np.ascontiguousarray(full[y0:y0 + CROP[0], x0:x0 + CROP[1]])
        k = ref_kernel(cfg)
        stats = {}
        if cfg.order is not None:
            out = fb.gpa_filter(crop, k, cfg.sigma_r, cfg.order, stats=stats)
            n = cfg.order
            method = "given"
        else:
            out, est = fb.gpa_filter_auto(crop, k, cfg.sigma_r, cfg.delta, stats=stats)
            n, method = est.N0, est.method
        exact = fb.bilateral_exact(crop, k, cfg.sigma_r)
        rep = fb.error_report(out, exact)
        arrays[f"{name}_in"] = crop
        arrays[f"{name}_out"] = out
        arrays[f"{name}_exact"] = exact
        scalars["cases"][name] = {
            "kind": cfg.kind, "sigma_s": cfg.sigma_s, "half_width": k.half_width, "sigma_r": cfg.sigma_r,
            "order": n, "order_method": method, "delta": cfg.delta, "w0": k.w0,
            "crop_origin": [y0, x0], "linf_vs_exact": rep.linf,
            "psnr_vs_exact": 20 * math.log10(255.0) - rep.mse_db,
            "spatial_filter_calls": stats["spatial_filter_calls"],
        }

    # ---- the reference's own engine test cases --------------------------------
    def case(tag, img, kind, param, sigma_r, order, allow=False, range_spec=None, with_exact=True):
        k = (fb.make_spatial_kernel("box", half_width=param) if kind == "box"
             else fb.make_spatial_kernel("gaussian", sigma_s=param))
        kw = {"allow_small_sigma": allow}
        if range_spec is not None:
            out = fb.gpa_filter(img, k, sigma_r, order, fb.RangeSpec(*range_spec), **kw)
        else:
            out = fb.gpa_filter(img, k, sigma_r, order, **kw)
        arrays[f"{tag}_in"] = np.asarray(img, np.float64)
        arrays[f"{tag}_out"] = out
        if with_exact:
            arrays[f"{tag}_exact"] = fb.bilateral_exact(img, k, sigma_r)
        scalars["cases"][tag] = {"kind": kind, "param": param, "sigma_r": sigma_r, "order": order,
                                 "allow_small_sigma": allow, "range_spec": range_spec}

    imp3 = np.zeros((3, 3)); imp3[1, 1] = 255.0
    case("impulse3", imp3, "box", 1, 50.0, 50)                       # test_engine.py:17-23
    imp5 = np.zeros((5, 5)); imp5[2, 2] = 255.0
    case("qdegenerate5", imp5, "box", 1, 10.0, 1, allow=True, with_exact=False)  # test_engine.py:112-119
    const = np.full((12, 12), 93.0)
    case("const_box", const, "box", 3, 40.0, 25)                     # test_engine.py:9-14
    case("const_gauss", const, "gaussian", 2, 40.0, 25)
    rng = np.random.default_rng(12345)
    r64 = np.floor(rng.uniform(0.0, 256.0, (64, 64)))
    case("random64_gauss5", r64, "gaussian", 5, 30.0, 60)            # test_engine.py:26-31
    rng = np.random.default_rng(7)
    r37 = np.floor(rng.uniform(0.0, 256.0, (37, 53)))
    case("ragged_box4", r37, "box", 4, 30.0, 30)
    case("ragged_gauss25", r37, "gaussian", 2.5, 30.0, 30)
    case("shift0_gauss2", r37 - 128.0, "gaussian", 2, 30.0, 40, range_spec=(128.0, 0.0))
    r8 = np.floor(np.random.default_rng(3).uniform(0.0, 256.0, (8, 8)))
    case("bigwindow_gauss5", r8, "gaussian", 5, 40.0, 20, with_exact=False)  # W=15 > dims: no window check
    row = np.floor(np.random.default_rng(4).uniform(0.0, 256.0, (1, 40)))
    case("row1x40_box2", row, "box", 2, 30.0, 20, with_exact=False)
    case("col40x1_gauss1", row.T.copy(), "gaussian", 1, 30.0, 20, with_exact=False)
    r48 = np.floor(np.random.default_rng(8).uniform(0.0, 256.0, (48, 48)))
    case("sigma12_box3", r48, "box", 3, 12.0, 120)                    # small sigma_r, large N

    # ---- spatial filters (conv.py) -----------------------------------------------
    rng = np.random.default_rng(99)
    s32 = np.floor(rng.uniform(0.0, 256.0, (32, 32)))
    arrays["spatial_in"] = s32
    for W in (1, 2, 7, 10):
        arrays[f"spatial_box{W}"] = fb.box_filter(s32, W)
    for s in (1.0, 3.0, 4.0):
        arrays[f"spatial_gauss{int(s)}"] = fb.gaussian_filter(s32, s)

    # ---- order selection ---------------------------------------------------------
    orders = []
    for sigma_r in range(10, 70):
        for eps in (1e-1, 1e-2, 1e-3, 1e-4, 1e-6):
            est = fb.estimate_order(float(sigma_r), eps, 128.0)
            orders.append([sigma_r, eps, est.N0, est.method,
                           est.newton_trace[0] if est.newton_trace else None])
    scalars["orders"] = orders
    scalars["epsilon_from_delta"] = [
        [d, w0, fb.epsilon_from_delta(d, w0, 128.0)]
        for d in (0.05, 0.1, 1.0, 3.0) for w0 in (1.0 / 9.0, 8.2645e-3, 6.3905e-3, 2.4977e-3)]

    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **arrays)
    with open(os.path.join(HERE, "reference_scalars.json"), "w") as fh:
        json.dump(scalars, fh, indent=1)
    print("wrote", len(arrays), "arrays,", len(scalars["cases"]), "cases")


if __name__ == "__main__":
    main()
