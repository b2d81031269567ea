"""ctypes binding of the C ABI in `include/fbgpu.h` (libfbgpu.so, built in-tree).

This is the only place the package touches native code.  There is no CPU
fallback: if the library is missing or no CUDA device is usable, every
filtering call raises `NativeError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import NativeError, NumericRangeError, ParameterError, RangeViolationError
from .image import range_message

LIB_NAME = "libfbgpu.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

FB_U8, FB_F32, FB_F64 = 0, 1, 2
FB_BOX, FB_GAUSSIAN = 0, 1
FB_PREC_F32, FB_PREC_F64 = 1, 2
(FB_OK, FB_ERR_PARAM, FB_ERR_NONFINITE_INPUT, FB_ERR_RANGE, FB_ERR_NUMERIC, FB_ERR_WINDOW,
 FB_ERR_CUDA, FB_ERR_NOMEM) = range(8)

#: Every symbol include/fbgpu.h declares (checked by tests/test_native_abi.py).
EXPORTED_SYMBOLS = (
    "fb_create", "fb_destroy", "fb_set_stream", "fb_set_workspace_limit", "fb_gpa_filter",
    "fb_gpa_filter_batch", "fb_spatial_filter", "fb_validate", "fb_bilateral_exact", "fb_last_error",
    "fb_version", "fb_launch_count", "fb_ipc_export", "fb_ipc_open", "fb_ipc_close", "fb_convolve_direct",
    "fb_error_stats", "fb_kernel_error_sup", "fb_build_id", "fb_gpa_filter_band",
)


class FbImage(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("on_device", ctypes.c_int32),
                ("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("ld", ctypes.c_int64)]


class FbSpatial(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("half_width", ctypes.c_int32),
                ("weights_1d", ctypes.POINTER(ctypes.c_double))]


class FbStats(ctypes.Structure):
    _fields_ = [("spatial_filter_calls", ctypes.c_int64), ("order", ctypes.c_int64),
                ("degenerate_pixels", ctypes.c_int64), ("nonfinite_outputs", ctypes.c_int64),
                ("bad_index", ctypes.c_int64), ("bad_value", ctypes.c_double),
                ("device_ms", ctypes.c_double), ("kernel_ms", ctypes.c_double),
                ("k1_ms", ctypes.c_double), ("k2_ms", ctypes.c_double),
                ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64),
                ("bands", ctypes.c_int32), ("precision", ctypes.c_int32), ("launches", ctypes.c_int64),
                ("bad_image", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None
_lib_lock = threading.Lock()
_contexts: dict[int, ctypes.c_void_p] = {}
# One lock per device context: a context (its workspace, flags, graphs) is not re-entrant
# (fbgpu.h), while ctypes releases the GIL during every call.
_ctx_locks: dict[int, threading.Lock] = {}


def load_library(path: str | None = None) -> ctypes.CDLL:
    """Load libfbgpu.so (once).  Raises NativeError when it has not been built."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        path = path or LIB_PATH
        if not os.path.exists(path):
            raise NativeError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        missing = [n for n in EXPORTED_SYMBOLS if not hasattr(lib, n)]
        if missing and path == LIB_PATH:
            raise NativeError(f"{path} lacks {', '.join(missing)}: stale build, rerun __graft_entry__.build()")
        if missing:  # an older A/B build: bind what it has
            class _Lib:
                def __init__(self, lib):
                    self._lib = lib

                def __getattr__(self, name):
                    try:
                        return getattr(self._lib, name)
                    except AttributeError:
                        return _Stub()

            class _Stub:
                argtypes = restype = None

                def __call__(self, *a):
                    raise NativeError("symbol missing from this A/B build")

            lib = _Lib(lib)
        P = ctypes.POINTER
        vp = ctypes.c_void_p
        lib.fb_create.argtypes = [ctypes.c_int, P(vp)]
        lib.fb_destroy.argtypes = [vp]
        lib.fb_set_stream.argtypes = [vp, vp]
        lib.fb_ipc_export.argtypes = [vp, ctypes.c_char_p, P(ctypes.c_int64)]
        lib.fb_ipc_open.argtypes = [ctypes.c_int32, ctypes.c_char_p, P(vp)]
        lib.fb_ipc_close.argtypes = [vp]
        lib.fb_set_workspace_limit.argtypes = [vp, ctypes.c_int64]
        lib.fb_gpa_filter.argtypes = [vp, P(FbImage), ctypes.c_int64, ctypes.c_int64, P(FbImage), P(FbSpatial),
                                      ctypes.c_double, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_int32, P(FbStats)]
        lib.fb_gpa_filter_band.argtypes = [vp, P(FbImage), P(FbImage), P(FbImage), ctypes.c_int64, ctypes.c_int64,
                                           P(FbImage), P(FbSpatial), ctypes.c_double, ctypes.c_int32,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_int32, P(FbStats)]
        lib.fb_gpa_filter_batch.argtypes = [vp, P(FbImage), P(FbImage), ctypes.c_int32, P(FbSpatial),
                                            ctypes.c_double, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_int32, P(FbStats)]
        lib.fb_spatial_filter.argtypes = [vp, P(FbImage), P(FbImage), P(FbSpatial), ctypes.c_int32, P(FbStats)]
        lib.fb_validate.argtypes = [vp, P(FbImage), ctypes.c_double, ctypes.c_double, P(FbStats)]
        lib.fb_bilateral_exact.argtypes = [vp, P(FbImage), P(FbImage), P(FbSpatial), ctypes.c_double, P(FbStats)]
        lib.fb_convolve_direct.argtypes = [vp, P(FbImage), P(FbImage), ctypes.c_int32, P(ctypes.c_double),
                                           P(FbStats)]
        lib.fb_error_stats.argtypes = [vp, P(FbImage), P(FbImage), P(ctypes.c_double), P(ctypes.c_double),
                                       P(FbStats)]
        lib.fb_kernel_error_sup.argtypes = [vp, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                            P(ctypes.c_double)]
        lib.fb_last_error.restype = ctypes.c_char_p
        lib.fb_version.restype = ctypes.c_int
        lib.fb_build_id.restype = ctypes.c_char_p
        if path == LIB_PATH:
            # the in-tree library must match the sources next to it (explicit paths are A/B variants)
            from ._buildid import source_build_id
            want, have = source_build_id(), lib.fb_build_id().decode()
            if want is not None and have != want:
                raise NativeError(f"{path} was built from other sources (build id {have}, sources {want}): "
                                  "rebuild with __graft_entry__.build()")
        lib.fb_launch_count.restype = ctypes.c_int64
        for name in ("fb_create", "fb_destroy", "fb_set_stream", "fb_set_workspace_limit", "fb_gpa_filter",
                     "fb_gpa_filter_band", "fb_gpa_filter_batch", "fb_spatial_filter", "fb_validate", "fb_bilateral_exact",
                     "fb_convolve_direct", "fb_error_stats", "fb_kernel_error_sup"):
            getattr(lib, name).restype = ctypes.c_int
        _lib = lib
        return lib


def context(device: int = 0) -> ctypes.c_void_p:
    """The per-device context (created on first use, owns the device workspace)."""
    lib = load_library()
    with _lib_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = ctypes.c_void_p()
            rc = lib.fb_create(device, ctypes.byref(ctx))
            if rc != FB_OK:
                raise NativeError(f"fb_create(device={device}) failed: {lib.fb_last_error().decode()}")
            _contexts[device] = ctx
            _ctx_locks[device] = threading.Lock()
        return ctx


def ctx_lock(device: int = 0) -> threading.Lock:
    """The lock serialising calls into the context of `device` (held around bind + call)."""
    context(device)
    return _ctx_locks[device]


def launch_count() -> int:
    return int(load_library().fb_launch_count())


def set_workspace_limit(nbytes: int, device: int = 0) -> None:
    lib = load_library()
    ctx = context(device)
    with _ctx_locks[device]:
        rc = lib.fb_set_workspace_limit(ctx, int(nbytes))
    _check(lib, rc, None, None)


# ----------------------------------------------------------------------------- arrays
_NP_DT = {np.dtype(np.uint8): FB_U8, np.dtype(np.float32): FB_F32, np.dtype(np.float64): FB_F64}
_TORCH_DT = {"torch.uint8": FB_U8, "torch.float32": FB_F32, "torch.float64": FB_F64}


def is_cuda_tensor(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def image_desc(arr) -> FbImage:
    """fb_image for a 2-D numpy array (host) or CUDA torch tensor (device); rows must be unit-stride.
    An FbImage passes through (e.g. a row slice of a peer's buffer, sharding.PeerOutput)."""
    if isinstance(arr, FbImage):
        return arr
    if is_cuda_tensor(arr):
        rs, cs = arr.stride()
        if cs != 1:
            raise ValueError("tensor rows must be contiguous")
        return FbImage(arr.data_ptr(), _TORCH_DT[str(arr.dtype)], 1, arr.shape[0], arr.shape[1], rs)
    isz = arr.itemsize
    if arr.shape[0] == 1:  # a single row: its row stride is irrelevant (numpy may report 0)
        return FbImage(arr.ctypes.data, _NP_DT[arr.dtype], 0, 1, arr.shape[1], arr.shape[1])
    if arr.strides[1] != isz or arr.strides[0] % isz or arr.strides[0] < arr.shape[1] * isz:
        raise ValueError("array rows must be contiguous")
    return FbImage(arr.ctypes.data, _NP_DT[arr.dtype], 0, arr.shape[0], arr.shape[1], arr.strides[0] // isz)


def ipc_export(dptr: int) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding dptr, offset of dptr in it)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    _check(lib, lib.fb_ipc_export(ctypes.c_void_p(dptr), buf, ctypes.byref(off)), None, None)
    return buf.raw, int(off.value)


def ipc_open(device: int, handle: bytes) -> int:
    """Map a peer allocation on `device`; returns its base address in this process."""
    lib = load_library()
    base = ctypes.c_void_p(0)
    _check(lib, lib.fb_ipc_open(int(device), ctypes.create_string_buffer(handle, 64), ctypes.byref(base)),
           None, None)
    return int(base.value)


def ipc_close(base: int) -> None:
    lib = load_library()
    _check(lib, lib.fb_ipc_close(ctypes.c_void_p(base)), None, None)


_spatial_cache: dict[int, tuple] = {}


def spatial_desc(kernel):
    """(FbSpatial, taps array keeping its pointer alive), cached per kernel object: the kernel is
    frozen, and rebuilding the ctypes descriptor is a measurable part of a small call."""
    hit = _spatial_cache.get(id(kernel))
    if hit is not None and hit[0] is kernel:
        return hit[1], hit[2]
    taps = np.ascontiguousarray(kernel.weights_1d, dtype=np.float64)
    kind = FB_BOX if kernel.kind == "box" else FB_GAUSSIAN
    desc = FbSpatial(kind, int(kernel.half_width), taps.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if len(_spatial_cache) >= 64:
        _spatial_cache.clear()
    _spatial_cache[id(kernel)] = (kernel, desc, taps)  # holds the kernel, so its id stays unique
    return desc, taps


def _check(lib, rc: int, src, stats: FbStats | None, lo=None, hi=None):
    """Translate a status code into the reference's exception (same classes and messages)."""
    if rc == FB_OK:
        return
    msg = lib.fb_last_error().decode(errors="replace")
    if rc == FB_ERR_NONFINITE_INPUT:
        raise ParameterError("image contains non-finite samples")
    if rc == FB_ERR_RANGE:
        cols = src.shape[1]
        row, col = divmod(int(stats.bad_index), cols)
        raise RangeViolationError(range_message(np.float64(stats.bad_value), row, col, lo, hi))
    if rc in (FB_ERR_PARAM, FB_ERR_WINDOW):
        raise ParameterError(msg)
    if rc == FB_ERR_NUMERIC:
        raise NumericRangeError(msg)
    raise NativeError(f"libfbgpu: {msg} (status {rc})")


_raw_stream = None
CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy (cuda_runtime_api.h)
_last_stream: dict[int, int | None] = {}  # context address -> stream last bound with fb_set_stream


def _stream_for(arr, device: int) -> int | None:
    """Raw cudaStream_t of torch's current stream on the tensor's device (None: the context's own)."""
    global _raw_stream
    if not is_cuda_tensor(arr):
        return None
    if _raw_stream is None:
        import torch
        getter = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        _raw_stream = getter if getter is not None else (
            lambda idx: torch.cuda.current_stream(idx).cuda_stream)
    s = _raw_stream(arr.device.index or 0)
    # torch's default stream is the legacy default stream (raw handle 0): bind it as
    # cudaStreamLegacy so the library orders its work after what torch queued there
    return CUDA_STREAM_LEGACY if not s else s


def _bind_stream(lib, ctx, stream: int | None) -> None:
    """fb_set_stream only when the stream differs from the one this context last used
    (small repeated calls are launch-bound: every skipped ctypes call is latency)."""
    key = ctx.value
    if _last_stream.get(key, -1) != stream:
        lib.fb_set_stream(ctx, ctypes.c_void_p(stream))
        _last_stream[key] = stream


def device_of(arr, device: int | None) -> int:
    if is_cuda_tensor(arr):
        return arr.device.index or 0
    return 0 if device is None else int(device)


def gpa(src, out, kernel, sigma_r: float, order: int, center: float, half_range: float, precision: int,
        device: int = 0, halo_top: int = 0, halo_bottom: int = 0) -> dict:
    """Run fb_gpa_filter; `src`/`out` are numpy arrays or CUDA tensors. Returns the stats dict."""
    lib = load_library()
    ctx = context(device)
    sp, _taps = spatial_desc(kernel)
    st = FbStats()
    with _ctx_locks[device]:
        _bind_stream(lib, ctx, _stream_for(src, device))
        rc = lib.fb_gpa_filter(ctx, ctypes.byref(image_desc(src)), halo_top, halo_bottom,
                               ctypes.byref(image_desc(out)), ctypes.byref(sp), float(sigma_r), int(order),
                               float(center), float(half_range), int(precision), ctypes.byref(st))
    _check(lib, rc, src, st, center - half_range, center + half_range)
    return st.as_dict()


def gpa_band(src, out, kernel, sigma_r: float, order: int, center: float, half_range: float, precision: int,
             row_origin: int, image_rows: int, above=None, below=None, device: int = 0) -> dict:
    """Run fb_gpa_filter_band: `src` = rows [row_origin, row_origin + rows) of an image_rows-row image,
    `above` / `below` = the neighbouring rows (CUDA tensors or FbImage views of a peer's buffer)."""
    lib = load_library()
    ctx = context(device)
    sp, _taps = spatial_desc(kernel)
    st = FbStats()
    ab = image_desc(above) if above is not None else None
    be = image_desc(below) if below is not None else None
    with _ctx_locks[device]:
        _bind_stream(lib, ctx, _stream_for(src, device))
        rc = lib.fb_gpa_filter_band(ctx, ctypes.byref(image_desc(src)), ctypes.byref(ab) if ab is not None else None,
                                    ctypes.byref(be) if be is not None else None, int(row_origin),
                                    int(image_rows), ctypes.byref(image_desc(out)), ctypes.byref(sp),
                                    float(sigma_r), int(order), float(center), float(half_range), int(precision),
                                    ctypes.byref(st))
    _check(lib, rc, src, st, center - half_range, center + half_range)
    return st.as_dict()


def gpa_batch(srcs, outs, kernel, sigma_r: float, order: int, center: float, half_range: float,
              precision: int, device: int = 0) -> dict:
    """Run fb_gpa_filter_batch over equally wide images (numpy arrays or CUDA tensors)."""
    lib = load_library()
    ctx = context(device)
    sp, _taps = spatial_desc(kernel)
    n = len(srcs)
    ins = (FbImage * n)(*[image_desc(s) for s in srcs])
    outs_d = (FbImage * n)(*[image_desc(o) for o in outs])
    st = FbStats()
    with _ctx_locks[device]:
        _bind_stream(lib, ctx, _stream_for(srcs[0], device))
        rc = lib.fb_gpa_filter_batch(ctx, ins, outs_d, n, ctypes.byref(sp), float(sigma_r), int(order),
                                     float(center), float(half_range), int(precision), ctypes.byref(st))
    bad = srcs[st.bad_image] if st.bad_image >= 0 else srcs[0]
    _check(lib, rc, bad, st, center - half_range, center + half_range)
    return st.as_dict()


def spatial(src, out, kernel, precision: int, device: int = 0) -> dict:
    lib = load_library()
    ctx = context(device)
    sp, _taps = spatial_desc(kernel)
    st = FbStats()
    with _ctx_locks[device]:
        _bind_stream(lib, ctx, _stream_for(src, device))
        rc = lib.fb_spatial_filter(ctx, ctypes.byref(image_desc(src)), ctypes.byref(image_desc(out)),
                                   ctypes.byref(sp), int(precision), ctypes.byref(st))
    _check(lib, rc, src, st)
    return st.as_dict()


def bilateral_exact(src, out, kernel, sigma_r: float, device: int = 0) -> dict:
    lib = load_library()
    ctx = context(device)
    sp, _taps = spatial_desc(kernel)
    st = FbStats()
    with _ctx_locks[device]:
        _bind_stream(lib, ctx, _stream_for(src, device))
        rc = lib.fb_bilateral_exact(ctx, ctypes.byref(image_desc(src)), ctypes.byref(image_desc(out)),
                                    ctypes.byref(sp), float(sigma_r), ctypes.byref(st))
    _check(lib, rc, src, st)
    return st.as_dict()


def validate(src, lo: float, hi: float, device: int = 0) -> None:
    """Device-side as_image finiteness + validate_range; raises like the reference."""
    lib = load_library()
    ctx = context(device)
    st = FbStats()
    with _ctx_locks[device]:
        _bind_stream(lib, ctx, _stream_for(src, device))
        rc = lib.fb_validate(ctx, ctypes.byref(image_desc(src)), float(lo), float(hi), ctypes.byref(st))
    _check(lib, rc, src, st, lo, hi)


def convolve_direct(src, out, weights_2d: np.ndarray, half_width: int, device: int = 0) -> dict:
    """fb_convolve_direct: the literal 2-D convolution with the (2W+1)^2 table (conv.py:83-96)."""
    lib = load_library()
    ctx = context(device)
    w2 = np.ascontiguousarray(weights_2d, dtype=np.float64)
    st = FbStats()
    with _ctx_locks[device]:
        _bind_stream(lib, ctx, _stream_for(src, device))
        rc = lib.fb_convolve_direct(ctx, ctypes.byref(image_desc(src)), ctypes.byref(image_desc(out)),
                                    int(half_width), w2.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                    ctypes.byref(st))
    _check(lib, rc, src, st)
    return st.as_dict()


def error_stats(a, b, device: int = 0) -> tuple[float, float]:
    """fb_error_stats: (max |a - b|, sum (a - b)^2) in fp64 on the device (analysis.py:33-46)."""
    lib = load_library()
    ctx = context(device)
    linf, ss = ctypes.c_double(0.0), ctypes.c_double(0.0)
    st = FbStats()
    with _ctx_locks[device]:
        _bind_stream(lib, ctx, _stream_for(a, device))
        rc = lib.fb_error_stats(ctx, ctypes.byref(image_desc(a)), ctypes.byref(image_desc(b)), ctypes.byref(linf),
                                ctypes.byref(ss), ctypes.byref(st))
    _check(lib, rc, a, st)
    return float(linf.value), float(ss.value)


def kernel_error_sup(order: int, sigma_r: float, half_range: float, device: int = 0) -> float:
    """fb_kernel_error_sup: grid supremum of the kernel error (analysis.py:70-103)."""
    lib = load_library()
    ctx = context(device)
    sup = ctypes.c_double(0.0)
    with _ctx_locks[device]:
        _bind_stream(lib, ctx, None)
        rc = lib.fb_kernel_error_sup(ctx, int(order), float(sigma_r), float(half_range), ctypes.byref(sup))
    _check(lib, rc, None, None)
    return float(sup.value)
