"""The C-ABI library loads and exports every symbol include/fbgpu.h declares (no GPU needed)."""

import ctypes
import os
import re

import pytest

from paper_1603_08109_b200 import _native

HEADER = os.path.join(os.path.dirname(__file__), "..", "include", "fbgpu.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|int64_t|void)\s+(fb_\w+)\s*\(", text, flags=re.M)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libfbgpu.so not built (run __graft_entry__.build())")
    lib = _native.load_library()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.fb_version() == 100


def test_struct_layouts():
    # int64-aligned C structs: sizes must match the header's field lists.
    assert ctypes.sizeof(_native.FbImage) == 8 + 4 + 4 + 8 * 3
    assert ctypes.sizeof(_native.FbSpatial) == 4 + 4 + 8
    assert ctypes.sizeof(_native.FbStats) == 8 * 12 + 4 + 4 + 8 + 8


def test_no_gpu_fails_loudly():
    """Without a CUDA device the product path raises instead of falling back to the CPU."""
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libfbgpu.so not built")
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    import numpy as np
    from paper_1603_08109_b200 import NativeError, gpa_filter, make_spatial_kernel
    with pytest.raises(NativeError):
        gpa_filter(np.zeros((8, 8)), make_spatial_kernel("box", half_width=1), 30.0, 5)


def test_stale_library_is_refused(monkeypatch):
    """The in-tree library carries the hash of the sources it was built from (fb_build_id); a
    library built from other sources must not load (a stale .so can never be the one that runs)."""
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libfbgpu.so not built (run __graft_entry__.build())")
    from paper_1603_08109_b200 import _buildid
    lib = _native.load_library()
    assert lib.fb_build_id().decode() == _buildid.source_build_id()
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_buildid, "source_build_id", lambda *a: "0123456789abcdef")
    with pytest.raises(_native.NativeError, match="other sources"):
        _native.load_library()
