"""Golden fixtures for the tools around the filter, from the REFERENCE itself.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_tools.py

Writes `tests/golden/reference_tools.npz` (arrays: PGM files the reference wrote, images it
loaded, convolve_direct outputs, CLI output rasters) and `tests/golden/reference_tools.json`
(scalars: kernel_error_sup, poisson_tail, psi_eval, accuracy_bound, order comparators,
range_kernel / gauss_poly, image-difference metrics, CLI reports and exit codes, I/O error
messages).  Tests only read the committed fixtures; the GPU box never runs this script.
"""

from __future__ import annotations

import json
import math
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
if os.path.isdir("/root/reference/pkg/src"):
    sys.path.insert(0, "/root/reference/pkg/src")

import fastbilateral as fb  # noqa: E402  (the reference)
from click.testing import CliRunner  # noqa: E402
from fastbilateral.cli import main as ref_cli  # noqa: E402

#: (N, sigma_r, T) grid-search cases: the reference tests' cases plus non-integer T and small grids
KERNEL_ERROR_CASES = [(1, 30.0, 128.0), (40, 30.0, 128.0), (20, 50.0, 128.0), (10, 70.0, 128.0),
                      (214, 10.0, 128.0), (300, 30.0, 128.0), (25, 50.0, 128.0), (5, 20.0, 37.5),
                      (60, 15.0, 100.0), (7, 40.0, 3.0), (33, 25.0, 128.0), (2, 100.0, 64.0)]


def rand_image(h, w, seed):
    return np.floor(np.random.default_rng(seed).uniform(0.0, 256.0, (h, w)))


def run_cli(args):
    res = CliRunner().invoke(ref_cli, args)
    return res.exit_code, res.output


def main():
    arrays: dict[str, np.ndarray] = {}
    sc: dict = {"reference_version": fb.__version__}
    tmp = tempfile.mkdtemp()

    # ---- PGM / PNG I/O (image.py:69-129) ------------------------------------------------
    edge = np.array([[-3.0, 0.49, 0.5, 254.5, 300.0, 127.5, 1.4999999999, 2.5000000001, 255.0, 0.0]])
    p = os.path.join(tmp, "edge.pgm")
    fb.save_pgm(p, edge)
    arrays["io_edge_in"] = edge
    arrays["io_edge_pgm"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
    img = np.random.default_rng(3).uniform(-20.0, 280.0, (13, 17))
    fb.save_pgm(p, img)
    arrays["io_rand_in"] = img
    arrays["io_rand_pgm"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
    headers = {
        "comment": b"P5\n# a comment\n2 2\n255\n\x00\x10\x20\xff",
        "multi_comment": b"P5 # c1\n# c2\n3 # w\n1\n# m\n255 \x01\x02\x03",
        "crlf_ws": b"P5\r\n2\t1 255\n\x07\x08",
    }
    for name, data in headers.items():
        p = os.path.join(tmp, name + ".pgm")
        open(p, "wb").write(data)
        arrays["io_hdr_" + name] = np.frombuffer(data, dtype=np.uint8)
        arrays["io_hdr_" + name + "_loaded"] = fb.load_pgm(p)
    bad = {"wrong_magic": b"P2\n2 2\n255\n0 0 0 0", "maxval": b"P5\n2 2\n65535\n\x00\x00\x00\x00",
           "no_dims": b"P5\n#only a comment\n", "garbage": b"not a pgm"}
    sc["io_errors"] = {}
    for name, data in bad.items():
        p = os.path.join(tmp, name + ".pgm")
        open(p, "wb").write(data)
        arrays["io_bad_" + name] = np.frombuffer(data, dtype=np.uint8)
        try:
            fb.load_pgm(p)
            sc["io_errors"][name] = None
        except ValueError as exc:
            sc["io_errors"][name] = str(exc).replace(p, "{path}")
    png_img = rand_image(9, 5, 11)
    p = os.path.join(tmp, "img.png")
    fb.save_image(p, png_img)
    arrays["io_png_bytes"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
    arrays["io_png_loaded"] = fb.load_image(p)

    # ---- convolve_direct (conv.py:83-96) ----------------------------------------------------
    conv_cases = {"box2": ((13, 17), "box", 2), "gauss15": ((20, 23), "gaussian", 1.5),
                  "row_box3": ((1, 29), "box", 3), "col_gauss1": ((31, 1), "gaussian", 1.0),
                  "box9_rect": ((40, 25), "box", 9)}
    sc["convolve_direct"] = {}
    for i, (name, (shape, kind, prm)) in enumerate(conv_cases.items()):
        im = rand_image(*shape, seed=100 + i)
        k = fb.make_spatial_kernel(kind, **({"half_width": prm} if kind == "box" else {"sigma_s": prm}))
        arrays["conv_" + name + "_in"] = im
        arrays["conv_" + name + "_out"] = fb.convolve_direct(im, k)
        sc["convolve_direct"][name] = {"kind": kind, "param": prm}

    # ---- metrology (analysis.py) -----------------------------------------------------------
    sc["kernel_error_sup"] = [[n, s, t, fb.kernel_error_sup(n, s, t)] for n, s, t in KERNEL_ERROR_CASES]
    sc["poisson_tail"] = [[n, lam, fb.poisson_tail(n, lam)]
                          for n in (0, 1, 5, 10, 40, 57, 100, 300) for lam in (0.5, 4.0, 18.2, 41.0, 163.8)]
    sc["psi_eval"] = [[s, n, sr, fb.psi_eval(s, n, sr)]
                      for s in (0.0, 1.0, 500.0, 16384.0) for n in (0, 1, 30) for sr in (30.0, 40.0)]
    sc["accuracy_bound"] = [[e, w0, t, fb.accuracy_bound(e, w0, t)]
                            for e in (0.0, 1e-6, 0.01) for w0 in (1.0 / 9.0, 6.39e-3, 1.0) for t in (128.0, 50.0)
                            if e < w0]
    a = rand_image(37, 41, 5)
    b = a + np.random.default_rng(6).normal(0.0, 0.3, a.shape)
    arrays["metric_a"], arrays["metric_b"] = a, b
    rep = fb.error_report(a, b)
    sc["metrics"] = {"linf": fb.linf_error(a, b), "mse_db": fb.mse_db(a, b), "linf_db": rep.linf_db}

    # ---- order comparators + range-kernel helpers (order.py, kernels.py) ------------------
    sc["chebyshev_order"] = [[lam, e, fb.chebyshev_order(lam, e).N0]
                             for lam in (0.5, 4.0, 18.2, 41.0, 163.8) for e in (1e-6, 1e-3, 0.1)]
    sc["order_approx"] = [[s, d, w0, t, fb.order_approx(s, d, w0, t).N0]
                          for s in (10.0, 30.0, 50.0, 69.0) for d in (0.1, 1.0) for w0 in (1 / 121, 6.39e-3)
                          for t in (128.0,)]
    sc["yang_order"] = [[s, d, fb.yang_order(s, d).N0] for s in (10.0, 20.0, 30.0, 50.0) for d in (0.1, 1.0, 3.0)]
    sc["range_kernel"] = [[t, s, float(fb.range_kernel(t, s))] for t in (0.0, 3.0, -50.0, 255.0)
                          for s in (10.0, 40.0)]
    sc["gauss_poly"] = [[t, tau, n, s, fb.gauss_poly(t, tau, n, s)]
                        for t, tau in ((0.0, 0.0), (10.0, -20.0), (128.0, 128.0), (-100.0, 77.0))
                        for n in (1, 5, 40) for s in (30.0, 50.0)]

    # ---- CLI (cli.py) -----------------------------------------------------------------------
    sc["cli"] = {}
    pgm24 = os.path.join(tmp, "in24.pgm")
    fb.save_pgm(pgm24, rand_image(24, 24, 21))
    arrays["cli_in24"] = np.frombuffer(open(pgm24, "rb").read(), dtype=np.uint8)
    # a 320 x 300 image (> 65,536 px, so the fp32 kernels run on our side)
    pgm_big = os.path.join(tmp, "big.pgm")
    fb.save_pgm(pgm_big, rand_image(320, 300, 22))
    arrays["cli_big"] = np.frombuffer(open(pgm_big, "rb").read(), dtype=np.uint8)
    filter_cases = {
        "gauss_delta": (pgm24, ["--spatial", "gaussian", "--sigma-s", "2", "--sigma-r", "50", "--delta", "0.1"]),
        "box_order": (pgm24, ["--spatial", "box", "--window", "3", "--sigma-r", "30", "--order", "40"]),
        "big_box_delta": (pgm_big, ["--spatial", "box", "--window", "5", "--sigma-r", "30", "--delta", "1"]),
        "big_gauss_order": (pgm_big, ["--spatial", "gaussian", "--sigma-s", "3", "--sigma-r", "40",
                                      "--order", "30"]),
    }
    for name, (src, opts) in filter_cases.items():
        out = os.path.join(tmp, name + ".pgm")
        rep = os.path.join(tmp, name + ".json")
        code, text = run_cli(["filter", src, out, *opts, "--report", rep])
        arrays["cli_filter_" + name] = np.frombuffer(open(out, "rb").read(), dtype=np.uint8)
        r = json.load(open(rep))
        arrays["cli_filter_" + name + "_float"] = (
            fb.gpa_filter_auto(fb.load_pgm(src), *_kernel_sigma(opts), float(_opt(opts, "--delta")))[0]
            if "--delta" in opts else
            fb.gpa_filter(fb.load_pgm(src), *_kernel_sigma(opts), int(_opt(opts, "--order"))))
        sc["cli"]["filter_" + name] = {"args": opts, "exit_code": code, "order": r["order"],
                                       "spatial_filter_calls": r["runtime_ms"]["spatial_filter_calls"]}
    ref_out = os.path.join(tmp, "ref.pgm")
    code, _ = run_cli(["reference", pgm24, ref_out, "--spatial", "box", "--window", "2", "--sigma-r", "30"])
    arrays["cli_reference_box2"] = np.frombuffer(open(ref_out, "rb").read(), dtype=np.uint8)
    sc["cli"]["reference_box2"] = {"exit_code": code}
    order_cases = {"eps": ["--sigma-r", "30", "--epsilon", "1e-3"],
                   "large_sigma": ["--sigma-r", "80", "--epsilon", "1e-3"],
                   "delta_gauss": ["--sigma-r", "30", "--delta", "0.1", "--spatial", "gaussian", "--sigma-s", "5"],
                   "delta_box": ["--sigma-r", "25", "--delta", "1", "--spatial", "box", "--window", "20"]}
    for name, opts in order_cases.items():
        rep = os.path.join(tmp, "o_" + name + ".json")
        code, text = run_cli(["order", *opts, "--report", rep])
        sc["cli"]["order_" + name] = {"args": opts, "exit_code": code, "report": json.load(open(rep)),
                                      "output": text}
    for name, opts in {"n40": ["--order", "40", "--sigma-r", "30"], "n300": ["--order", "300", "--sigma-r", "30"],
                       "n10_t50": ["--order", "10", "--sigma-r", "20", "--t", "50"]}.items():
        rep = os.path.join(tmp, "k_" + name + ".json")
        code, text = run_cli(["kernel-error", *opts, "--report", rep])
        sc["cli"]["kernel_error_" + name] = {"args": opts, "exit_code": code, "report": json.load(open(rep))}
    cmp_cases = {"box_order20": ["--spatial", "box", "--window", "2", "--sigma-r", "30", "--order", "20"],
                 "gauss_delta": ["--spatial", "gaussian", "--sigma-s", "2", "--sigma-r", "50", "--delta", "0.1"]}
    for name, opts in cmp_cases.items():
        rep = os.path.join(tmp, "c_" + name + ".json")
        code, text = run_cli(["compare", pgm24, *opts, "--report", rep])
        r = json.load(open(rep))
        sc["cli"]["compare_" + name] = {"args": opts, "exit_code": code, "errors": r["errors"], "order": r["order"]}
    usage = {"both": ["filter", pgm24, "o.pgm", "--spatial", "box", "--window", "2", "--sigma-r", "30",
                      "--delta", "1", "--order", "10"],
             "neither": ["filter", pgm24, "o.pgm", "--spatial", "box", "--window", "2", "--sigma-r", "30"],
             "no_sigma_s": ["filter", pgm24, "o.pgm", "--spatial", "gaussian", "--sigma-r", "30", "--order", "10"],
             "small_sigma": ["filter", pgm24, "o.pgm", "--spatial", "box", "--window", "2", "--sigma-r", "5",
                             "--order", "10"],
             "window_too_big": ["filter", pgm24, "o.pgm", "--spatial", "box", "--window", "30", "--sigma-r", "30",
                                "--order", "10"],
             "range": ["filter", pgm24, "o.pgm", "--spatial", "box", "--window", "2", "--sigma-r", "30",
                       "--order", "10", "--t", "10"],
             "order_no_spatial": ["order", "--sigma-r", "30", "--delta", "1"],
             "kernel_error_n0": ["kernel-error", "--order", "0", "--sigma-r", "30"]}
    sc["cli"]["exit_codes"] = {}
    for name, args in usage.items():
        args = [a if a != "o.pgm" else os.path.join(tmp, "o.pgm") for a in args]
        code, text = run_cli(args)
        sc["cli"]["exit_codes"][name] = {"args": [a.replace(tmp, "{tmp}") for a in args], "exit_code": code,
                                         "output": text.replace(tmp, "{tmp}")}

    np.savez_compressed(os.path.join(HERE, "reference_tools.npz"), **arrays)
    with open(os.path.join(HERE, "reference_tools.json"), "w") as fh:
        json.dump(sc, fh, indent=1, default=float)
        fh.write("\n")
    print("wrote", len(arrays), "arrays")


def _opt(opts, name):
    return opts[opts.index(name) + 1]


def _kernel_sigma(opts):
    if _opt(opts, "--spatial") == "box":
        k = fb.make_spatial_kernel("box", half_width=int(_opt(opts, "--window")))
    else:
        k = fb.make_spatial_kernel("gaussian", sigma_s=float(_opt(opts, "--sigma-s")))
    return k, float(_opt(opts, "--sigma-r"))


if __name__ == "__main__":
    main()
