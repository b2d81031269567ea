"""Summarise ncu captures into profiles/ (committed evidence).

  python tools/ncu_summary.py full  gpurun_out/prof_c4.ncu-rep  --config c4 --pixels 67108864 --out profiles/ncu_c4.json
  python tools/ncu_summary.py launches gpurun_out/launches_c4.csv --out profiles/r01_launches_c4.md

`full`: per kernel of a `--set full` report: duration, DRAM bytes read/written
(per launch), achieved DRAM bandwidth, FMA-pipe and issue utilisation, warp
occupancy and the top stall reasons.  `--pixels` = output pixels per launch,
so bytes/pixel can be compared with the algorithmic bytes in DESIGN.md.
`launches`: the per-launch device times of a `--metrics gpu__time_duration.sum`
run, aggregated by kernel (count, total, share).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_ld_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
}
SCALE = {"dram__bytes_read.sum": {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0},
         "dram__bytes_write.sum": {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0},
         "gpu__time_duration.sum": {"msecond": 1e3, "ms": 1e3, "usecond": 1.0, "us": 1.0, "nsecond": 1e-3,
                                    "ns": 1e-3, "second": 1e6, "s": 1e6}}


def _num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def full(rep: str, config: str, pixels: float | None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").split("<")[0].strip().split("::")[-1]
        d = {"kernel": name}
        for key, metric in METRICS.items():
            if metric not in hdr:
                continue
            i = hdr.index(metric)
            v = _num(r[i])
            if v is not None and metric in SCALE:
                v *= SCALE[metric].get(units[i], 1.0)
            d[key] = v
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                v = _num(r[i])
                if v:
                    stalls.append((v, h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(v for v, _ in stalls) or 1.0
        d["top_stalls_pct"] = {h: round(100 * v / tot, 1) for v, h in sorted(stalls, reverse=True)[:6]}
        traffic = (d.get("dram_read_bytes") or 0) + (d.get("dram_write_bytes") or 0)
        d["dram_bytes_per_launch"] = traffic
        if d.get("duration_us"):
            d["dram_gbs"] = traffic / (d["duration_us"] * 1e-6) / 1e9
            d["dram_frac_of_measured_peak"] = d["dram_gbs"] / 6542.7
        if pixels:
            d["dram_bytes_per_output_pixel"] = traffic / pixels
        kernels.setdefault(short, d)  # first capture of each kernel
    return {"config": config, "report": rep, "pixels_per_launch": pixels, "kernels": kernels,
            "note": "ncu --set full --clock-control none: cold-cache, serialised replays; compare shares, "
                    "not absolute times, with bench.py's CUDA-event timings"}


def launches(path: str):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = _num(r[vi]) or 0.0
        v *= SCALE["gpu__time_duration.sum"].get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    total = sum(t for _, t in agg.values()) or 1.0
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{name}` | {n} | {t:.1f} | {100 * t / total:.1f}% |")
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["full", "launches"])
    ap.add_argument("path")
    ap.add_argument("--config", default="")
    ap.add_argument("--pixels", type=float, default=None)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    if a.mode == "full":
        out = json.dumps(full(a.path, a.config, a.pixels), indent=1)
    else:
        out = launches(a.path)
    with open(a.out, "w") as fh:
        fh.write(out)
    print(out[:3000])


if __name__ == "__main__":
    sys.exit(main())
