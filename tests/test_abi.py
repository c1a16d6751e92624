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
