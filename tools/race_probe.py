"""Race probe (compute-sanitizer is closed on this GPU pool): every kernel family is run
repeatedly on the same inputs, alternately alone and next to a second stream that saturates HBM
with copies (timing perturbation), and every output must be bit-identical to the first run.
A stage-ring or staging-buffer race (a tile overwritten while still read, a row stored before it
is complete) changes outputs from run to run; round 1's proxy-fence race was found this way.

  python tools/race_probe.py [--reps 10] > gpurun_out/race_probe.txt
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_08109_b200 import _native, make_spatial_kernel, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()

noise_a = torch.empty(1 << 28, dtype=torch.float32, device="cuda")  # 1 GiB each
noise_b = torch.empty_like(noise_a)
noise_stream = torch.cuda.Stream()


def contend(n=6):
    with torch.cuda.stream(noise_stream):
        for _ in range(n):
            noise_b.copy_(noise_a)


def kern(kind, p):
    return make_spatial_kernel(kind, **({"half_width": p} if kind == "box" else {"sigma_s": p}))


# (label, image shape, input dtype, kind, W or sigma_s, sigma_r, N, precision)
CASES = [
    ("tile box W=5 (c1)", (1024, 1024), np.float32, "box", 5, 50.0, 10, _native.FB_PREC_F32),
    ("tile box W=16 f64", (600, 700), np.float32, "box", 16, 25.0, 30, _native.FB_PREC_F64),
    ("tile gauss W=9 (c0) f64 in", (512, 512), np.float64, "gaussian", 3.0, 40.0, 15, _native.FB_PREC_F32),
    ("tile gauss W=15 (c2)", (1024, 2048), np.float32, "gaussian", 5.0, 30.0, 42, _native.FB_PREC_F32),
    ("tile gauss W=24 (c3)", (1024, 1024), np.float32, "gaussian", 8.0, 20.0, 76, _native.FB_PREC_F32),
    ("tile gauss W=32", (700, 900), np.float32, "gaussian", 32 / 3, 20.0, 60, _native.FB_PREC_F32),
    ("gauss W=9 f64", (700, 900), np.float32, "gaussian", 3.0, 20.0, 40, _native.FB_PREC_F64),
    ("walker W=20 N=57 (c4)", (2048, 4096), np.float32, "box", 20, 25.0, 57, _native.FB_PREC_F32),
    ("walker W=1 N=63", (2048, 2100), np.float32, "box", 1, 25.0, 63, _native.FB_PREC_F32),
    ("walker W=32 N=7 u8 in", (2048, 2100), np.uint8, "box", 32, 60.0, 7, _native.FB_PREC_F32),
    ("walker f64 W=20 N=57", (2048, 2100), np.float32, "box", 20, 25.0, 57, _native.FB_PREC_F64),
    ("generic W=40 box", (600, 700), np.float32, "box", 40, 25.0, 20, _native.FB_PREC_F32),
]

t0 = time.time()
bad = 0
for label, shape, dt, kind, p, sr, N, prec in CASES:
    img = synth.config_image("c4", height=shape[0], width=shape[1])
    img = np.floor(img).astype(dt) if dt == np.uint8 else img.astype(dt)
    d = torch.from_numpy(img).cuda()
    k = kern(kind, p)
    outs = [torch.empty(shape, dtype=torch.float64, device="cuda") for _ in range(args.reps)]
    for i, o in enumerate(outs):  # distinct outputs: eager calls (no graph replay)
        if i % 2:
            contend()
        _native.gpa(d, o, k, sr, N, 128.0, 128.0, prec, 0)
    torch.cuda.synchronize()
    first = outs[0].cpu().numpy()
    diffs = [float(np.max(np.abs(o.cpu().numpy() - first))) for o in outs[1:]]
    ok = all(x == 0.0 for x in diffs) and np.all(np.isfinite(first))
    bad += not ok
    print(f"{'OK  ' if ok else 'FAIL'} {label:28s} {args.reps} runs ({args.reps // 2} under HBM contention), "
          f"max run-to-run |d| {max(diffs):.3g}", flush=True)
    del outs, d
print(f"race_probe: {len(CASES) - bad}/{len(CASES)} kernel families bit-stable in {time.time() - t0:.1f}s")
sys.exit(1 if bad else 0)
