"""The C-ABI library loads, exports exactly what include/pcbz_b200.h declares,
and refuses to compute without a device (no CPU fallback).  CPU only."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2310_09467_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "pcbz_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^PCBZ_API\s+[\w\s\*]*?\b(pcbz_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "pcbz_residual_bwt_pair_hist" in syms and "pcbz_judge_device" in syms
    assert len(syms) >= 19


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_binding_table_matches_header():
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_version_and_error_plumbing():
    assert "sm_100a" in _lib.version()
    assert isinstance(_lib.device_count(), int)


@pytest.mark.skipif(_lib.device_count() > 0, reason="only meaningful on a host without a GPU")
def test_no_silent_cpu_fallback():
    from paper_2310_09467_b200 import _kernels
    img = np.arange(12, dtype=np.uint16).reshape(3, 4)
    with pytest.raises(RuntimeError):
        _kernels.residual_bwt_pair_hist(img, 1, 1, 1)


def test_missing_library_fails_loudly(tmp_path):
    import importlib
    saved = _lib._lib
    try:
        _lib._lib = None
        with pytest.raises(ImportError):
            _lib.load(tmp_path / "nope.so")
    finally:
        _lib._lib = saved


def test_sm100a_cubin_present():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_native_join_equals_bytes_join():
    """_lib.join (pcbz_gather, the device coder's container join) is b"".join
    for bytes, memoryviews into numpy buffers and empty parts, multithreaded
    once the total is large."""
    rng = np.random.default_rng(7)
    big = rng.integers(0, 256, 24 << 20, dtype=np.uint8)
    mv = memoryview(big)
    parts = [b"PCBZ", b"", mv[5:5 + (9 << 20)], bytes(rng.integers(0, 256, 1000, dtype=np.uint8)),
             mv[(9 << 20) + 11:], b"x", mv[0:0]]
    assert _lib.join(parts, threads=8) == b"".join(parts)
    assert _lib.join([], threads=4) == b""
    small = [bytes([i]) * i for i in range(50)]
    assert _lib.join(small, threads=3) == b"".join(small)


def test_gather_rejects_bad_pieces():
    lib = _lib.load()
    dst = np.zeros(8, np.uint8)
    lens = np.array([4, -1], np.int64)
    srcs = (ctypes.c_void_p * 2)(dst.ctypes.data, dst.ctypes.data)
    assert lib.pcbz_gather(dst.ctypes.data, srcs, lens.ctypes.data, 2, 2) == _lib.PCBZ_E_INVALID


def test_temporal_undelta_inverts_the_delta():
    from paper_2310_09467_b200 import Frame, LensletGeometry, temporal_undelta
    rng = np.random.default_rng(9)
    geo = LensletGeometry(3, 3)
    cur = rng.integers(0, 65536, (17, 11), dtype=np.uint16)
    prev = rng.integers(0, 65536, (17, 11), dtype=np.uint16)
    delta = ((cur.astype(np.int32) - prev.astype(np.int32)) % 65536).astype(np.uint16)
    assert np.array_equal(temporal_undelta(Frame(delta, geo), Frame(prev, geo)).samples, cur)
