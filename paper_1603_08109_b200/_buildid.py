"""Build identity of libfbgpu.so: a hash of the CUDA/C sources and the compile flags.

`__graft_entry__.build()` compiles it into the library (`fb_build_id()`), and
`_native.load_library()` refuses a library whose id differs from the sources next to it,
so a stale `.so` (older sources, other flags) can never be the one that runs.
"""

from __future__ import annotations

import hashlib
import os

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")

NVCC_FLAGS = (
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    # no --use_fast_math / -ftz: the Q-floor test needs fp32 values down to ~1e-36
)


def source_files() -> list[str]:
    out = []
    for d in (CSRC, INCLUDE):
        if os.path.isdir(d):
            out += sorted(os.path.join(d, f) for f in os.listdir(d) if f.endswith((".cu", ".cuh", ".h")))
    return out


def source_build_id(extra_flags: tuple[str, ...] = ()) -> str | None:
    """16 hex digits over every source file (name + bytes) and the flags; None without sources."""
    files = source_files()
    if not files:
        return None
    h = hashlib.sha256()
    for p in files:
        h.update(os.path.basename(p).encode() + b"\0")
        with open(p, "rb") as fh:
            h.update(fh.read())
        h.update(b"\0")
    h.update(" ".join(NVCC_FLAGS + tuple(extra_flags)).encode())
    return h.hexdigest()[:16]
