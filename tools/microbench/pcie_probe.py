"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently (CUDA events), to bound e2e.

  python tools/microbench/pcie_probe.py
"""
import torch

GiB = 1 << 30
h_in = torch.empty(GiB, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(2 * GiB, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(GiB, dtype=torch.uint8, device="cuda")
d_out = torch.empty(2 * GiB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"H2D 1 GiB: {t1:.2f} ms = {GiB / t1 / 1e6:.1f} GB/s")
print(f"D2H 2 GiB: {t2:.2f} ms = {2 * GiB / t2 / 1e6:.1f} GB/s")
print(f"H2D 1 GiB || D2H 2 GiB: {t3:.2f} ms  (c4 e2e transfer floor: {268435456 / t3 / 1e3:.0f} MP/s)")
