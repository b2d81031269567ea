"""Benchmark of the GPA bilateral filter hot path (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

A "step" is one pass of the filter over the config's whole workload:
  c4 (default): one 16384^2 float32 image, box W=20, sigma_r=25, delta=1 -> N=57;
                at N>1 GPUs: row bands (starts at multiples of 256 rows) whose kernel 1 reads
                the neighbours' halo rows in place and whose kernel 2 writes into rank 0's
                output (CUDA IPC; no collective).
  c3: 64 float32 images of 2048^2, Gaussian sigma_s=8, sigma_r=20, delta=1 -> N=76; by image.
  c0/c1/c2: single images (replicas at N>1).
`value` = megapixels/s over all ranks with inputs resident in HBM (device
events, max over ranks); `e2e` = the same metric through the public API with
host buffers (H2D of the input and D2H of the float64 result inside the timed
region).  Inputs are larger than L2 (126 MB) for c2-c4 and the channel
workspace is several GB, so no L2 flush is needed there; c0/c1 flush L2
between steps.  `--impl reference` times the CPU restatement of the
reference algorithm (oracle/, numpy fp64) on all host cores instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1603_08109_b200 import synth  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
FP32_NOMINAL_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4; FFMA probe measured 72-74 (profiles/)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-legs", action="store_true",
                    help="skip the fp64 leg and the per-config device legs of the other configs")
    ap.add_argument("--cpu-sample-mp", type=float, default=0.0, help="override the CPU sample size (MP)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def peaks():
    try:
        with open(PEAKS_FILE) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every ~5 ms through NVML while the timed
    region runs (a short timed region still gets samples; nvidia-smi -lms takes ~0.3 s to start).
    The timed region starts only after the first sample has been taken."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, cuda_index: int):
        self.cuda_index = cuda_index
        self.samples = []  # (sm_mhz, reasons bitmask)
        self.max_mhz = None
        self._stop = threading.Event()
        self.error = None

    def __enter__(self):
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda._get_nvml_device_index(self.cuda_index))
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
            t0 = time.monotonic()
            while not self.samples and time.monotonic() - t0 < 1.0:
                time.sleep(0.001)
        except Exception as e:  # no NVML: the line says so (samples = 0)
            self.error = repr(e)
            self.h = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)),
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))))
            except Exception as e:
                self.error = repr(e)
                return
            time.sleep(0.005)

    def __exit__(self, *exc):
        self._stop.set()
        if self.h is not None:
            self.thread.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0, "error": self.error}
        reasons = set()
        for _, bits in self.samples:
            for name, const in self.REASONS:
                if bits & getattr(self.nv, const, 0):
                    reasons.add(name)
        sm = [m for m, _ in self.samples]
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(np.min(sm)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm), "source": "NVML, 5 ms"}


def algorithmic_bytes(cfg, N, ch_bytes=4):
    """Per pixel: B_alg = 2 s_io + 2 (N+1) s_ch and the split over the two kernels
    (s_ch = 4 for the fp32 planes, 8 for the fp64 path's planes)."""
    s_in = np.dtype(cfg.dtype).itemsize
    s_out = 4  # device-resident runs write float32
    ch = (N + 1) * ch_bytes
    return {"pipeline": s_in + s_out + 2 * ch, "k1": s_in + ch, "k2": ch + s_in + s_out}


def algorithmic_flops(cfg, N):
    """FP32 FLOPs per pixel of the two kernels (FMA = 2): taps per pass x channels + Horner."""
    W = synth.config_kernel(cfg).half_width
    if cfg.kind == "box":
        per_pass = 2  # running sum: one add, one subtract
    else:
        per_pass = 2 * (2 * W + 1)
    return {"k1": (N + 1) * (per_pass + 2), "k2": (N + 1) * (per_pass + 6)}


def ncu_traffic(config, stage):
    """(kernel name, dram bytes per launch) of pipeline stage 'k1'/'k2' from the committed ncu
    summary of this config (profiles/ncu_<config>.json, tools/ncu_summary.py), else (None, None)."""
    path = os.path.join(ROOT, "profiles", f"ncu_{config}.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        prefix = {"fused": "k_small"}.get(stage, stage)  # the small-image kernel is k_small_fused
        for name, k in d["kernels"].items():
            if name.startswith(prefix):
                return name, k["dram_bytes_per_launch"], d.get("pixels_per_launch")
    except Exception:
        pass
    return None, None, None


# ----------------------------------------------------------------------------- reference arm (CPU)
_CPU_IMG = None  # shared with forked workers (no per-job pickling of the image)


def _oracle_tile(args):
    y0, y1, x0, x1, kind, W, taps, sigma_r, N = args
    from oracle import gpa_oracle
    img = _CPU_IMG
    H, Wd = img.shape
    ya, yb, xa, xb = max(0, y0 - W), min(H, y1 + W), max(0, x0 - W), min(Wd, x1 + W)
    out = gpa_oracle.gpa(img[ya:yb, xa:xb], kind, W, taps, sigma_r, N)
    return out[y0 - ya:y1 - ya, x0 - xa:x1 - xa]


def cpu_sample_region(cfg, target_mp):
    """A contiguous block of the workload of about `target_mp` megapixels (whole rows of image 0)."""
    rows = max(64, min(cfg.height, int(target_mp * 1e6 / cfg.width)))
    return rows, cfg.width


def run_cpu(img, cfg, N, rows, cores):
    """Filter the first `rows` rows of `img` with the oracle on `cores` processes; returns seconds."""
    k = synth.config_kernel(cfg)
    tile_r = 256
    tile_c = min(cfg.width, 2048)
    global _CPU_IMG
    _CPU_IMG = np.ascontiguousarray(img[: min(cfg.height, rows + k.half_width)])
    jobs = []
    for y in range(0, rows, tile_r):
        for x in range(0, cfg.width, tile_c):
            jobs.append((y, min(rows, y + tile_r), x, min(cfg.width, x + tile_c), cfg.kind,
                         k.half_width, k.weights_1d, cfg.sigma_r, N))
    t0 = time.perf_counter()
    if cores > 1:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(cores) as pool:
            pool.map(_oracle_tile, jobs, chunksize=1)
    else:
        for j in jobs:
            _oracle_tile(j)
    return time.perf_counter() - t0


def host_info() -> dict:
    """The CPU the baselines ran on (core count, model, thread variables)."""
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            model = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), "")
    except OSError:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(),
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
            "FASTBILATERAL_THREADS": os.environ.get("FASTBILATERAL_THREADS")}


def reference_arm(args, cfg, N):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    img = synth.config_image(cfg)
    # ~2 MP per core per step keeps a step near 10 s on one of these Xeons.
    per_core_mp = 2.0 if cfg.kind == "box" else 0.8
    target = args.cpu_sample_mp or per_core_mp * cores
    rows, cols = cpu_sample_region(cfg, target)
    mp_per_step = rows * cols / 1e6
    for _ in range(args.warmup):
        run_cpu(img, cfg, N, rows, cores)
    times = [run_cpu(img, cfg, N, rows, cores) for _ in range(args.steps)]
    total = sum(times)
    value = mp_per_step * args.steps / total
    sample = (f"first {rows} rows x {cols} cols of image 0 ({mp_per_step:.2f} MP) per step, "
              f"tiled 256x2048 with W halos over a {cores}-process pool; numpy fp64 oracle/gpa_oracle.py")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (paper_1603_08109_b200/synth.py, seeded)", "config": config_block(cfg, N, args.gpus),
        "cpu_baseline": {"value": value, "unit": "MP/s", "cores": cores, "kind": "port", "sample": sample,
                         "host": host_info()},
        "e2e": {"value": value, "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "megapixels/sec (order N, per spatial kind) at 1/2/4/8 B200; % of HBM roofline"


def config_block(cfg, N, world):
    k = synth.config_kernel(cfg)
    par = ("by-image" if cfg.batch > 1 else ("row-bands" if cfg.name == "c4" else "replicas")) + f" x{world}"
    l2 = "inputs+workspace > L2 (126 MB), no flush" if cfg.pixels * 4 > 126e6 else "L2 flushed between steps"
    return {"workload": cfg.name, "image": [cfg.batch, cfg.height, cfg.width], "input_dtype": cfg.dtype,
            "spatial": cfg.kind, "half_width": k.half_width, "sigma_s": cfg.sigma_s, "sigma_r": cfg.sigma_r,
            "order_N": N, "delta": cfg.delta, "parallelism": par, "l2": l2}


# ----------------------------------------------------------------------------- our arm (GPU)
def _gen_image(args):
    cfg_name, index = args
    return synth.config_image(synth.CONFIGS[cfg_name], index)


def config_images(cfg, indices):
    """The seeded synthetic images `indices` of a config, generated on all host cores."""
    indices = list(indices)
    if len(indices) <= 2:
        return [synth.config_image(cfg, i) for i in indices]
    import multiprocessing as mp
    with mp.get_context("fork").Pool(min(len(indices), os.cpu_count() or 1)) as pool:
        return pool.map(_gen_image, [(cfg.name, i) for i in indices])


def kernel_roofline(cfg, N, per_launch_ms, px_per_launch, launches, step_ms_total, ch_bytes=4):
    """Per-kernel achieved HBM GB/s and FP32 TFLOP/s (algorithmic bytes / flops per launch over
    the launch's CUDA-event time) and the dominant kernel's bound and fraction of peak."""
    hbm_peak, _ = peaks()
    bpp = algorithmic_bytes(cfg, N, ch_bytes)
    fpp = algorithmic_flops(cfg, N)
    kernels = {}
    if per_launch_ms["k2"] <= 0:
        # small images: one fused kernel (fb_small.cuh), no channel planes in HBM; its algorithmic
        # bytes are the input and the output only, its flops those of both passes
        t = per_launch_ms["k1"] * 1e-3
        s_io = bpp["k1"] + bpp["k2"] - (bpp["pipeline"])  # = s_in (counted twice in k1 + k2)
        b = bpp["pipeline"] - 2 * (bpp["k1"] - s_io)      # s_in + s_out
        f = fpp["k1"] + fpp["k2"]
        kernels["fused"] = {
            "avg_launch_ms": t * 1e3,
            "share_of_step": per_launch_ms["k1"] * launches / max(1e-9, step_ms_total),
            "hbm_gbs": b * px_per_launch / t / 1e9,
            "hbm_frac": b * px_per_launch / t / 1e9 / hbm_peak,
            "fp32_tflops": f * px_per_launch / t / 1e12,
            "fp32_frac": f * px_per_launch / t / 1e12 / FP32_NOMINAL_TFLOPS,
            "alg_bytes_per_px": b,
            "two_kernel_alg_bytes_per_px": bpp["pipeline"],
        }
        dk = kernels["fused"]
        return kernels, "fused", "hbm" if dk["hbm_frac"] >= dk["fp32_frac"] else "fp32"
    for name in ("k1", "k2"):
        t = per_launch_ms[name] * 1e-3
        kernels[name] = {
            "avg_launch_ms": t * 1e3,
            "share_of_step": per_launch_ms[name] * launches / max(1e-9, step_ms_total),
            "hbm_gbs": bpp[name] * px_per_launch / t / 1e9,
            "hbm_frac": bpp[name] * px_per_launch / t / 1e9 / hbm_peak,
            "fp32_tflops": fpp[name] * px_per_launch / t / 1e12,
            "fp32_frac": fpp[name] * px_per_launch / t / 1e12 / FP32_NOMINAL_TFLOPS,
            "alg_bytes_per_px": bpp[name],
        }
    dom = max(("k1", "k2"), key=lambda n: per_launch_ms[n])
    dk = kernels[dom]
    bound = "hbm" if dk["hbm_frac"] >= dk["fp32_frac"] else "fp32"
    return kernels, dom, bound


def eager_kernel_times(native, imgs, like, kernel, cfg, N, precision, device, calls):
    """Per-kernel CUDA-event times from eager calls (each into a fresh output buffer: a new
    CUDA-graph key, so the call launches kernel by kernel with its events)."""
    import torch
    k1 = k2 = 0.0
    nl = 0
    fresh = [torch.empty_like(like) for _ in range(calls)]
    for i, o in enumerate(fresh):
        st = native.gpa(imgs[i % len(imgs)], o, kernel, cfg.sigma_r, N, 128.0, 128.0, precision, device)
        k1, k2, nl = k1 + st["k1_ms"], k2 + st["k2_ms"], nl + max(1, st["bands"])
    return {"k1": k1 / nl, "k2": k2 / nl}


def device_leg(cfg, N, steps, warmup, device, precision, imgs=None):
    """One rank's device-resident timed steps of a config (inputs in HBM, float32 output), L2
    flushed between steps when the workload fits L2.  Returns value / timing / roofline."""
    import torch

    from paper_1603_08109_b200 import _native
    dev = torch.device("cuda", device)
    kernel = synth.config_kernel(cfg)
    if imgs is None:
        imgs = [torch.from_numpy(im).to(dev) for im in config_images(cfg, range(cfg.batch))]
    outs = [torch.empty(im.shape, dtype=torch.float32, device=dev) for im in imgs]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if cfg.pixels * 4 <= 126e6 else None
    stream = torch.cuda.current_stream(dev)

    def step():
        if len(imgs) > 1:
            return _native.gpa_batch(imgs, outs, kernel, cfg.sigma_r, N, 128.0, 128.0, precision, device)
        return _native.gpa(imgs[0], outs[0], kernel, cfg.sigma_r, N, 128.0, 128.0, precision, device)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    ev, sts = [], []
    for _ in range(steps):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sts.append(step())
        b.record(stream)
        ev.append((a, b))
    torch.cuda.synchronize(dev)
    ms = sum(a.elapsed_time(b) for a, b in ev)
    launches = sum(st["bands"] for st in sts)  # per kernel: one launch of each per row band
    k1 = sum(st["k1_ms"] for st in sts)
    k2 = sum(st["k2_ms"] for st in sts)
    if k1 < 0 or k2 < 0 or len(imgs) > 1:
        # graph replays time only the whole call; a batch overlaps two streams: take the split
        # from eager one-image calls on one stream outside the timed region
        per_launch = eager_kernel_times(_native, imgs, outs[0], kernel, cfg, N, precision, device, max(2, steps))
        split_from = "eager one-image calls outside the timed region"
    else:
        per_launch = {"k1": k1 / launches, "k2": k2 / launches}
        split_from = "timed steps (CUDA events per kernel)"
    px = sum(int(im.shape[0]) * int(im.shape[1]) for im in imgs)
    px_per_launch = px * steps / launches
    kernels, dom, bound = kernel_roofline(cfg, N, per_launch, px_per_launch, launches, ms,
                                          8 if precision == _native.FB_PREC_F64 else 4)
    hbm_peak, _ = peaks()
    bpp = algorithmic_bytes(cfg, N, 8 if precision == _native.FB_PREC_F64 else 4)
    del outs, flush
    return {"value": px * steps / (ms * 1e-3) / 1e6, "unit": "MP/s", "ms_per_step": ms / steps, "steps": steps,
            "warmup": warmup, "ms_total": ms, "launches_per_kernel": launches, "kernels": kernels,
            "dominant": dom, "bound": bound,
            "frac": kernels[dom]["hbm_frac"] if bound == "hbm" else kernels[dom]["fp32_frac"],
            "pipeline_hbm_frac": bpp["pipeline"] * px * steps / (ms * 1e-3) / 1e9 / hbm_peak,
            "kernel_times_from": split_from, "pixels_per_step": px}


def main():
    args = parse()
    cfg = synth.CONFIGS[args.config]
    N = synth.config_order(cfg)
    if args.impl == "reference":
        reference_arm(args, cfg, N)
        return

    import torch
    import torch.distributed as dist

    from paper_1603_08109_b200 import _native, gpa_filter, gpa_filter_batch, sharding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    kernel = synth.config_kernel(cfg)
    W = kernel.half_width

    # ---- this rank's share of the workload (host copies kept for e2e) --------------------
    bands = None
    host_ext = None
    if cfg.batch > 1:
        idx = list(sharding.image_shard(cfg.batch, world, rank))
        host_imgs = config_images(cfg, idx)
    else:
        full = synth.config_image(cfg)
        if world > 1 and cfg.name == "c4":
            bands = sharding.RowBands(cfg.height, world, W)
            r0, r1 = bands.bounds(rank)
            host_imgs = [np.ascontiguousarray(full[r0:r1])]
            e0, e1 = bands.extended_bounds(rank)
            host_ext = np.ascontiguousarray(full[e0:e1])  # the band with its halo rows (e2e leg)
        else:
            host_imgs = [full]
        del full
    dev_imgs = [torch.from_numpy(im).to(dev) for im in host_imgs]
    dev_out = [torch.empty(im.shape, dtype=torch.float32, device=dev) for im in host_imgs]
    my_pixels = sum(im.shape[0] * im.shape[1] for im in host_imgs)
    root_full = None
    peer = pin = None
    if bands is not None:
        # no collective on the data path: kernel 1 reads the W halo rows in place from the
        # neighbours' input bands (sharding.PeerInput, CUDA IPC over NVLink / NVSwitch), and the
        # final gather is fused into kernel 2, which writes every rank's rows straight into the
        # root's buffer (sharding.PeerOutput); the hand-offs are store flags
        if rank == 0:
            root_full = torch.empty((cfg.height, cfg.width), dtype=torch.float32, device=dev)
        peer = sharding.PeerOutput(root_full, (cfg.height, cfg.width), torch.float32, rank, local)
        pin = sharding.PeerInput(dev_imgs[0], bands, rank, local)
        torch.cuda.synchronize(dev)
        pin.publish()  # the inputs are written once: one hand-off before the steps
        pin.wait_neighbours()
    flush = None
    if cfg.pixels * 4 <= 126e6:
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    ctx_stream = torch.cuda.current_stream(dev)
    kstats = {"k1_ms": 0.0, "k2_ms": 0.0, "kernel_ms": 0.0, "calls": 0, "launches": 0, "bands": 0}

    def step(record=False):
        if bands is not None:
            r0, r1 = bands.bounds(rank)
            st = _native.gpa_band(dev_imgs[0], peer.band(r0, r1), kernel, cfg.sigma_r, N, 128.0, 128.0,
                                  _native.FB_PREC_F32, row_origin=r0, image_rows=cfg.height, above=pin.above,
                                  below=pin.below, device=local)
            sts = [st]
            peer.done()
        elif len(dev_imgs) > 1:
            sts = [_native.gpa_batch(dev_imgs, dev_out, kernel, cfg.sigma_r, N, 128.0, 128.0,
                                     _native.FB_PREC_F32, local)]
        else:
            sts = [_native.gpa(dev_imgs[0], dev_out[0], kernel, cfg.sigma_r, N, 128.0, 128.0,
                               _native.FB_PREC_F32, local)]
        if record:
            for st in sts:
                kstats["k1_ms"] += st["k1_ms"]
                kstats["k2_ms"] += st["k2_ms"]
                kstats["kernel_ms"] += st["kernel_ms"]
                kstats["calls"] += 1
                kstats["launches"] += st["launches"]
                kstats["bands"] += st["bands"]

    def timed(fn, steps):
        ev = []
        for _ in range(steps):
            if flush is not None:
                flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(ctx_stream)
            fn()
            e.record(ctx_stream)
            ev.append((s, e))
        torch.cuda.synchronize(dev)
        return sum(s.elapsed_time(e) for s, e in ev)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    n_launch0 = _native.launch_count()
    with ClockSampler(local) as clocks:
        ms = timed(lambda: step(record=True), args.steps)
    launches = _native.launch_count() - n_launch0
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    total_px = cfg.pixels  # every rank's share together is the whole workload
    value = total_px * args.steps / (ms_max * 1e-3) / 1e6

    # ---- e2e through the public API with host buffers ------------------------------------
    e2e = None
    if not args.no_e2e:
        # row bands (N > 1): each rank's host input is its band plus the halo rows, filtered
        # through the C ABI's band entry point (bit-identical rows to a one-GPU call)
        e2e_in = [host_ext] if host_ext is not None else host_imgs
        pinned_in = [torch.from_numpy(im).pin_memory().numpy() for im in e2e_in]
        pinned_out = [torch.empty(im.shape, dtype=torch.float64).pin_memory().numpy() for im in host_imgs]

        e2e_st = {}  # the library's own count of the bytes each call moved over PCIe

        def e2e_step():
            if len(pinned_in) > 1:
                gpa_filter_batch(pinned_in, kernel, cfg.sigma_r, N, precision="f32", device=local, outs=pinned_out,
                                 stats=e2e_st)
            else:
                if host_ext is not None:
                    top, bottom = bands.halos(rank)
                    r0, r1 = bands.bounds(rank)
                    ext = pinned_in[0]
                    e2e_st.update(_native.gpa_band(
                        ext[top:top + r1 - r0], pinned_out[0], kernel, cfg.sigma_r, N, 128.0, 128.0,
                        _native.FB_PREC_F32, row_origin=r0, image_rows=cfg.height,
                        above=ext[:top] if top else None, below=ext[top + r1 - r0:] if bottom else None,
                        device=local))
                else:
                    gpa_filter(pinned_in[0], kernel, cfg.sigma_r, N, precision="f32", device=local,
                               out=pinned_out[0], stats=e2e_st)

        for _ in range(max(1, args.warmup)):  # the device leg's warm-up (small calls turn into
            t_w = time.perf_counter()          # CUDA-graph replays after the first sightings)
            e2e_step()
            t_w = time.perf_counter() - t_w
        # at least K calls, and enough of them to span ~0.2 s of host clock (sub-ms calls)
        n_e2e = max(1, args.steps, min(4000, int(0.2 / max(t_w, 1e-6))))
        if world > 1:
            n_t = torch.tensor([n_e2e], dtype=torch.int64, device=dev)
            dist.all_reduce(n_t, op=dist.ReduceOp.MAX)
            n_e2e = int(n_t.item())
            dist.barrier()
        # Each call is synchronous (H2D, kernels, D2H on the context stream), so the
        # host clock around the calls is the end-to-end time.
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            e2e_step()
        t_ms = (time.perf_counter() - t0) * 1e3
        t_t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_t, op=dist.ReduceOp.MAX)
        e2e = {"value": total_px * n_e2e / (float(t_t.item()) * 1e-3) / 1e6, "unit": "MP/s",
               "h2d_bytes_per_step": int(e2e_st.get("h2d_bytes", sum(im.nbytes for im in pinned_in))) * world,
               "d2h_bytes_per_step": int(e2e_st.get("d2h_bytes", sum(o.nbytes for o in pinned_out))) * world,
               "host_out_bytes_per_step": int(sum(o.nbytes for o in pinned_out)) * world,
               "calls": n_e2e,
               "path": ("gpa_filter_batch" if len(pinned_in) > 1 else "gpa_filter")
               + f"(pinned {pinned_in[0].dtype} numpy in, out= pinned float64 numpy): H2D, kernels and D2H pipelined "
                 "inside the call; byte counts are the library's (calls over 16 MP send the fp32 path's float32 "
                 "centred result over PCIe and widen it to the float64 output on host threads, "
                 "csrc/fb_hostwiden.cuh)"
               + ("; at N>1 each rank filters its band from host memory through fb_gpa_filter_band with its "
                  "halo rows (libfbgpu C ABI), output rows to its own pinned buffer" if bands is not None else "")}
        del pinned_in, pinned_out

    if peer is not None:
        dist.barrier()  # teardown: every rank is done with the peer mappings before unmapping
        peer.close()
        pin.close()
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel --------------------------------------------------
    hbm_peak, peak_src = peaks()
    bpp = algorithmic_bytes(cfg, N)
    launches_per_kernel = max(1, kstats["bands"])  # one launch of each kernel per row band
    kernel_times_from = "timed steps (CUDA events per kernel)"
    per_launch = {n: kstats[f"{n}_ms"] / launches_per_kernel for n in ("k1", "k2")}  # ms
    if kstats["k1_ms"] < 0 or kstats["k2_ms"] < 0 or len(dev_imgs) > 1:
        # graph replays (fbgpu.h: k1_ms = k2_ms = -1) time only the whole call, and a timed
        # batch alternates two streams (overlapping per-kernel spans): split from eager
        # one-image calls on one stream outside the timed region
        per_launch = eager_kernel_times(_native, dev_imgs, dev_out[0], kernel, cfg, N, _native.FB_PREC_F32,
                                        local, max(2, args.steps))
        kernel_times_from = "eager one-image calls outside the timed region"
    px_per_launch = my_pixels * args.steps / launches_per_kernel
    kernels, dom, bound = kernel_roofline(cfg, N, per_launch, px_per_launch, launches_per_kernel, ms)
    dk = kernels[dom]
    kname, traffic, traffic_px = ncu_traffic(cfg.name, dom)
    if traffic is not None and traffic_px and abs(traffic_px - px_per_launch) > 1:
        traffic = traffic * px_per_launch / traffic_px  # profile captured on a different launch size
    roofline = {
        "bound": bound, "kernel": kname or dom,
        "achieved": dk["hbm_gbs"] if bound == "hbm" else dk["fp32_tflops"],
        "peak": hbm_peak if bound == "hbm" else FP32_NOMINAL_TFLOPS,
        "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
        "frac": dk["hbm_frac"] if bound == "hbm" else dk["fp32_frac"],
        "traffic": traffic,
        "traffic_source": "profiles/ncu_%s.json (ncu --set full, dram__bytes_read+write per launch)" % cfg.name
        if traffic is not None else None,
        "peak_source": peak_src if bound == "hbm" else "nominal 148 SM x 128 FMA/clk x 1.965 GHz",
        "alg_bytes_per_px": dk["alg_bytes_per_px"],
        "pipeline_hbm_frac": bpp["pipeline"] * total_px * args.steps / (ms_max * 1e-3) / 1e9 / hbm_peak,
        "kernels": kernels,
        "kernel_times_from": kernel_times_from,
    }

    # ---- same-precision (fp64) leg and the other configs, device-resident, rank 0, N = 1 ----
    f64 = per_config = None
    if world == 1 and not args.no_extra_legs:
        del dev_out
        torch.cuda.empty_cache()
        # the fp64 path (the reference's arithmetic type) on the same inputs
        leg = device_leg(cfg, N, max(2, min(args.steps, 5)), max(1, min(args.warmup, 2)), local,
                         _native.FB_PREC_F64, dev_imgs)
        f64 = {k: leg[k] for k in ("value", "unit", "ms_per_step", "steps", "dominant", "bound", "frac",
                                   "pipeline_hbm_frac")}
        f64["dtype"] = "f64"
        f64["k1_ms"], f64["k2_ms"] = leg["kernels"]["k1"]["avg_launch_ms"], leg["kernels"]["k2"]["avg_launch_ms"]
        f64["note"] = "precision='f64': fp64 channel planes and arithmetic throughout (8 B per plane value)"
        del dev_imgs
        torch.cuda.empty_cache()
        per_config = {}
        for name in sorted(synth.CONFIGS):
            if name == cfg.name:
                continue
            c = synth.CONFIGS[name]
            leg = device_leg(c, synth.config_order(c), args.steps, args.warmup, local, _native.FB_PREC_F32)
            per_config[name] = {"value": leg["value"], "unit": "MP/s", "ms_per_step": leg["ms_per_step"],
                                "steps": leg["steps"], "order_N": synth.config_order(c), "dominant": leg["dominant"],
                                "bound": leg["bound"], "frac": leg["frac"],
                                "pipeline_hbm_frac": leg["pipeline_hbm_frac"],
                                "k1_ms": leg["kernels"]["k1"]["avg_launch_ms"],
                                "k2_ms": leg["kernels"]["k2"]["avg_launch_ms"],
                                "kernel_times_from": leg["kernel_times_from"],
                                "config": config_block(c, synth.config_order(c), 1)}
            torch.cuda.empty_cache()

    # ---- CPU baseline (rank 0, N=1 only, bounded sample, one core) ------------------------
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        img0 = host_imgs[0] if cfg.batch > 1 or bands is None else synth.config_image(cfg)
        target = args.cpu_sample_mp or (2.5 if cfg.kind == "box" else 1.0)
        rows, cols = cpu_sample_region(cfg, target)
        secs = run_cpu(img0, cfg, N, rows, 1)
        cpu = {"value": rows * cols / 1e6 / secs, "unit": "MP/s", "cores": 1, "kind": "port",
               "sample": f"first {rows} rows x {cols} cols of image 0 ({rows * cols / 1e6:.2f} MP), numpy fp64 "
                         f"restatement of the reference (oracle/gpa_oracle.py), one process",
               "host": host_info()}

    line = {
        "metric": METRIC, "value": value, "unit": "MP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (paper_1603_08109_b200/synth.py, seeded; BASELINE recipes)",
        "config": config_block(cfg, N, world), "clocks": clocks.summary(), "gpu_launches": launches,
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "f64": f64, "per_config": per_config,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
