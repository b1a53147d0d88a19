"""CPU: the C-ABI library loads, exports every symbol include/curvalign_cuda.h
declares, validates arguments like the reference, and fails loudly (never falls
back to the CPU) when no CUDA device is present. No kernel is launched here."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2501_17779_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "curvalign_cuda.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cva_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 12
    lib = ctypes.CDLL(_native.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in curvalign_cuda.h but not exported"
    # the Python binding covers every declared symbol
    assert set(syms) == set(_native.SIGNATURES)


def test_abi_version_and_struct_layout():
    lib = _native.load()
    assert lib.cva_abi_version() == 1
    assert ctypes.sizeof(_native.cva_alignment) == 48
    assert np.dtype(_native.ALIGNMENT_DTYPE).itemsize == 48


def test_argument_validation_without_device():
    lib = _native.load()
    z = np.zeros((1, 3, 2))
    # N < 4 -> invalid_argument (proj/src/rigid_align.cpp:18-21), checked before any device work
    assert lib.cva_align_batch_host(z.ctypes.data, z.ctypes.data, 1, 3, 0, 0) == _native.CVA_INVALID_ARGUMENT
    # n_out < 8 -> invalid_argument (proj/src/curve.cpp:69)
    offs = np.array([0, 3], dtype=np.int64)
    pts = np.zeros((3, 2))
    assert lib.cva_preprocess_batch(pts.ctypes.data, offs.ctypes.data, 1, 3, 4, 1, pts.ctypes.data, 0, None) \
        == _native.CVA_INVALID_ARGUMENT
    # SRV needs >= 8 nodes (proj/src/srv.cpp:72)
    assert lib.cva_srv_align_batch_host(z.ctypes.data, z.ctypes.data, 1, 4, 0, 0) == _native.CVA_INVALID_ARGUMENT
    # curve buffers are double2 arrays: 8-byte-aligned pointers are rejected before any launch
    buf = np.zeros(8 * 64 + 2)
    base = buf.ctypes.data + (8 if buf.ctypes.data % 16 == 0 else 0)  # an odd multiple of 8
    out = np.zeros(1, dtype=_native.ALIGNMENT_DTYPE)
    assert lib.cva_align_batch(base, base, 1, 64, out.ctypes.data, None, None) == _native.CVA_INVALID_ARGUMENT
    assert b"16-byte aligned" in lib.cva_last_error()
    assert lib.cva_preprocess_align_batch(base, offs.ctypes.data, 1, 3, 1024, 1, out.ctypes.data, None, None) \
        == _native.CVA_INVALID_ARGUMENT


@pytest.mark.skipif(_native.load().cva_device_count() > 0, reason="a CUDA device is present")
def test_no_device_fails_loudly():
    lib = _native.load()
    c = np.zeros((1, 64, 2))
    out = np.zeros(1, dtype=_native.ALIGNMENT_DTYPE)
    rc = lib.cva_align_batch_host(c.ctypes.data, c.ctypes.data, 1, 64, out.ctypes.data, 0)
    assert rc == _native.CVA_CUDA_ERROR
    assert b"CUDA" in lib.cva_last_error()
    from paper_2501_17779_b200 import align_fft

    with pytest.raises(_native.CurvalignError):
        align_fft(np.random.default_rng(0).standard_normal((64, 2)), np.zeros((64, 2)))


def test_python_errors_mirror_reference():
    from paper_2501_17779_b200 import align_fft, preprocess

    with pytest.raises(ValueError):  # size mismatch (rigid_align.cpp:19)
        align_fft(np.zeros((32, 2)), np.zeros((64, 2)))
    with pytest.raises(ValueError):  # n_out < 8 (curve.cpp:69)
        preprocess(np.zeros((16, 2)), 4)
