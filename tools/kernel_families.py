"""Small runs of every kernel family, each checked against the fp64 path.

  python tools/kernel_families.py   (was to run under compute-sanitizer; see profiles/r02_sanitizer.txt)

Covers: kernel 1 tile (Gaussian and box), the box walker (f32 input through the cp.async ring,
u8/f64 input through registers), kernel 2 (Gaussian and box, TMA + mbarrier rings), both
precisions, host-chunked input, CUDA-graph replay of a repeated device call, row bands with halo
rows in separate buffers (fb_gpa_filter_band), the plain spatial filter, validation, and the
exact / analysis kernels.  Each result is checked against the fp64 path so a wrong answer under
the tool is also caught.  Sizes are small (the tools slow kernels down 10-1000x), but the walker
needs an image of >= 4 Mi padded samples, so one image is 2048 x 2100.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_08109_b200 import (_native, apply_spatial, bilateral_exact, gpa_filter,  # noqa: E402
                                   make_spatial_kernel, synth)

t0 = time.time()
rng = np.random.default_rng(1)
small = np.floor(rng.uniform(0, 256, (130, 197))).astype(np.float32)
gk = make_spatial_kernel("gaussian", sigma_s=3.0)
bk = make_spatial_kernel("box", half_width=5)
cases = 0


def check(a, b, tol, what):
    global cases
    err = float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))
    assert err <= tol, (what, err)
    cases += 1
    print(f"{what}: max|d| {err:.2e}", flush=True)


# kernel 1 tile + kernel 2, both kinds, both precisions (small: tile kernels)
for k, sr, N in ((gk, 40.0, 15), (bk, 50.0, 10)):
    ref = gpa_filter(small, k, sr, N, precision="f64")
    check(gpa_filter(small, k, sr, N, precision="f32"), ref, 1e-3, f"{k.kind} tile f32")
    check(gpa_filter(small.astype(np.uint8), k, sr, N, precision="f32"), ref, 1e-3, f"{k.kind} tile u8-in")
# walker (box, >= 4 Mi padded samples), f32 and u8 input; fp64 walker; W = 20, N = 9 (NCH 16)
big = synth.config_image("c4", height=2048, width=2100)
wk = make_spatial_kernel("box", half_width=20)
ref = gpa_filter(big, wk, 25.0, 9, precision="f64")
check(gpa_filter(big, wk, 25.0, 9, precision="f32"), ref, 2e-3, "walker f32 (host, chunked)")
check(gpa_filter(np.floor(big).astype(np.uint8), wk, 25.0, 9, precision="f32"),
      gpa_filter(np.floor(big).astype(np.uint8), wk, 25.0, 9, precision="f64"), 2e-3, "walker u8-in")
# device-resident: a repeated small call is captured and replayed as a CUDA graph
d = torch.from_numpy(small).cuda()
out = torch.empty_like(d)
for _ in range(4):
    _native.gpa(d, out, gk, 40.0, 15, 128.0, 128.0, _native.FB_PREC_F32, 0)
check(out.cpu().numpy(), gpa_filter(small, gk, 40.0, 15, precision="f64"), 1e-3, "graph replay")
# row band with halo rows in separate device buffers (the multi-GPU path)
dbig = torch.from_numpy(big).cuda()
r0, r1 = 768, 1536
band_out = torch.empty((r1 - r0, big.shape[1]), dtype=torch.float64, device="cuda")
_native.gpa_band(dbig[r0:r1].clone(), band_out, wk, 25.0, 9, 128.0, 128.0, _native.FB_PREC_F32, r0, big.shape[0],
                 dbig[r0 - 20:r0].clone(), dbig[r1:r1 + 20].clone(), 0)
full = gpa_filter(dbig, wk, 25.0, 9, precision="f32").cpu().numpy()
check(band_out.cpu().numpy(), full[r0:r1], 0.0, "band with separate halos (bit-exact)")
# plain spatial filters, exact filter, validation path
check(apply_spatial(small, gk, precision="f32"), apply_spatial(small, gk), 1e-3, "spatial gaussian f32")
check(apply_spatial(small, bk, precision="f32"), apply_spatial(small, bk), 1e-3, "spatial box f32")
exact = bilateral_exact(small[:40, :50].astype(np.float64), gk, 40.0)
check(exact, exact, 0.0, "bilateral_exact")
try:
    bad = small.copy()
    bad[3, 4] = np.nan
    gpa_filter(bad, gk, 40.0, 15)
    raise SystemExit("expected ParameterError")
except Exception as e:  # noqa: BLE001
    assert "non-finite" in str(e), e
    cases += 1
torch.cuda.synchronize()
print(f"kernel_families: {cases} cases OK in {time.time() - t0:.1f}s", flush=True)
