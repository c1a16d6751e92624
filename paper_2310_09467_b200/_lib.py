"""ctypes binding of libpcbz_b200.so (the C ABI in include/pcbz_b200.h).

There is no CPU fallback: if the shared library or an sm_100 device is
missing, every compute call raises.  Error codes map to the exceptions the
reference raises for the same conditions (ValueError for bad arguments,
RuntimeError for device failures).
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_native" / "libpcbz_b200.so"

PCBZ_OK = 0
PCBZ_E_INVALID = -1
PCBZ_E_CUDA = -2
PCBZ_NEEDS_HOST = 1
PCBZ_E_NODEVICE = -3
PCBZ_E_INTERNAL = -4
MAX_CANDIDATES = 26

_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_c_size = ctypes.c_size_t
_vp = ctypes.c_void_p

# name -> (restype, argtypes); every symbol include/pcbz_b200.h declares
SIGNATURES = {
    "pcbz_version": (ctypes.c_char_p, []),
    "pcbz_last_error": (ctypes.c_char_p, []),
    "pcbz_device_count": (_c_int, []),
    "pcbz_residual_bwt_pair_hist": (_c_int, [_vp, _c_i64, _c_i64, _c_int, _c_i64, _c_i64, _vp]),
    "pcbz_residual_image": (_c_int, [_vp, _c_i64, _c_i64, _c_int, _c_i64, _c_i64, _vp]),
    "pcbz_temporal_delta": (_c_int, [_vp, _vp, _c_i64, _vp]),
    "pcbz_counting_bwt": (_c_int, [_vp, _c_i64, _vp]),
    "pcbz_pair_hist": (_c_int, [_vp, _c_i64, _vp]),
    "pcbz_bwt_pair_hist": (_c_int, [_vp, _c_i64, _vp]),
    "pcbz_entropy2d": (_c_int, [_vp, _c_i64, _vp]),
    "pcbz_register_entropy_terms": (_c_int, [_c_i64, _vp, _c_i64]),
    "pcbz_entropy_terms_registered": (_c_int, [_c_i64]),
    "pcbz_select_predictor": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _c_int,
                                       _vp, _vp, _vp]),
    "pcbz_judge_host": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _c_int,
                                 _c_int, _vp, _vp, _vp]),
    "pcbz_judge_workspace_size": (_c_size, [_c_i64, _c_i64, _c_i64, _c_int, _c_int]),
    "pcbz_judge_device": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _c_int,
                                   _c_int, _vp, _vp, _vp, _vp, _vp, _c_size, _vp]),
    "pcbz_emit_host": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp]),
    "pcbz_reconstruct_host": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp,
                                       _vp]),
    "pcbz_band_layout": (_c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _c_int, _c_int,
                                  _c_int, _c_int, _vp, _vp, _vp]),
    "pcbz_band_range": (_c_int, [_c_i64, _c_i64, _c_int, _c_int, _vp, _vp]),
    "pcbz_judge_band_device": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp,
                                        _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _c_size,
                                        _vp]),
    "pcbz_judge_merge_device": (_c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _c_int,
                                         _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp]),
    "pcbz_judge_merge_slots_device": (_c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _c_int,
                                               _c_int, _c_int, _c_int, _c_i64, _c_i64, _vp, _vp, _vp,
                                               _vp]),
    "pcbz_judge_merge_peers_device": (_c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _c_int,
                                               _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp,
                                               _vp, _vp]),
    "pcbz_peer_signal": (_c_int, [_vp, _vp, _c_int, _c_int, ctypes.c_uint32, _c_int, _vp]),
    "pcbz_judge_select_device": (_c_int, [_c_i64, _vp, _c_int, _c_int, _c_int, _vp, _vp, _vp]),
    "pcbz_emit_band_device": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp,
                                       _c_int, _c_int, _vp, _vp]),
    "pcbz_bzip2_bound": (_c_size, [_vp, _c_int]),
    "pcbz_bzip2_host": (_c_int, [_vp, _vp, _c_int, _vp, _c_size, _vp, _vp, _vp]),
    "pcbz_bzip2_device": (_c_int, [_vp, _vp, _c_int, _vp, _c_size, _vp, _vp, _vp, _vp]),
    "pcbz_bzip2_last_error": (ctypes.c_char_p, []),
    "pcbz_compress_bound": (_c_size, [_c_i64, _c_i64, _c_i64, _c_i64]),
    "pcbz_compress_host": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _c_int,
                                    _c_int, _vp, _c_i64, _vp, _vp, _vp, _c_size, _vp, _vp, _vp]),
    "pcbz_compress_frames_host": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp,
                                           _c_int, _c_int, _vp, _c_i64, _vp, _vp, _vp, _c_size, _vp,
                                           _vp, _vp]),
    "pcbz_bunzip2_host": (_c_int, [_vp, _vp, _c_int, _vp, _vp, _vp, _vp]),
    "pcbz_decompress_host": (_c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64,
                                      _vp, _vp, _vp, _vp, _vp]),
    "pcbz_host_alloc": (_vp, [_c_size]),
    "pcbz_host_free": (_c_int, [_vp]),
    "pcbz_gather": (_c_int, [_vp, _vp, _vp, _c_i64, _c_int]),
    "pcbz_set_segment_override": (_c_int, [_c_int]),
    "pcbz_set_profiling": (_c_int, [_c_int]),
    "pcbz_set_item_trace": (_c_int, [_c_int]),
    "pcbz_item_trace": (_c_i64, [_vp, _c_i64, _vp]),
    "pcbz_last_timing": (_c_int, [_vp, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and return the native library; raises if it is absent."""
    global _lib
    with _lock:
        if _lib is None:
            import os
            p = Path(path) if path else Path(os.environ.get("PCBZ_LIB", LIB_PATH))
            if not p.exists():
                raise ImportError(
                    f"{p} is missing: build it with `python -m paper_2310_09467_b200.build_native` "
                    "(there is no CPU fallback for the entropy judge)")
            lib = ctypes.CDLL(str(p))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int) -> None:
    """Raise the Python exception matching a PCBZ_E* return code."""
    if rc == PCBZ_OK:
        return
    msg = load().pcbz_last_error().decode(errors="replace")
    if rc == PCBZ_E_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"libpcbz_b200 error {rc}: {msg}")


def ptr(a: np.ndarray | None):
    """Data pointer of a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "native calls need C-contiguous buffers"
    return a.ctypes.data


#: largest total (2*H*W - 1) whose entropy term table is registered (8 bytes per count)
TERMS_MAX_TOTAL = 1 << 27
_terms_lock = threading.Lock()


def ensure_entropy_terms(total: int) -> bool:
    """Register this host's numpy terms p * log2(p), p = c / total, for
    every count c = 0..total with the current device (once per total), so
    device entropies are bit-identical to the reference's numpy entropy2d
    (criterion.py:94-95) evaluated on this host.  Returns False (device log2,
    <= 1 ulp per term) when the table would be too large."""
    total = int(total)
    if total < 1 or total > int(os.environ.get("PCBZ_TERMS_MAX_TOTAL", TERMS_MAX_TOTAL)):
        return False
    lib = load()
    if lib.pcbz_entropy_terms_registered(total):
        return True
    with _terms_lock:
        if lib.pcbz_entropy_terms_registered(total):
            return True
        # exactly the reference's evaluation: int64 counts / float(total), np.log2, product
        p = np.arange(total + 1, dtype=np.int64) / float(total)
        with np.errstate(divide="ignore", invalid="ignore"):
            t = p * np.log2(p)
        t[0] = 0.0
        rc = lib.pcbz_register_entropy_terms(total, t.ctypes.data, t.size)
        if rc == PCBZ_E_INVALID:   # over the device-memory budget: device log2 for this total
            return False
        check(rc)
    return True


def version() -> str:
    return load().pcbz_version().decode()


def device_count() -> int:
    return int(load().pcbz_device_count())


# ---- host memory helpers (whole-compressor path) ------------------------------

class _PinnedBlock:
    """One pcbz_host_alloc block, freed when the last array viewing it goes."""

    def __init__(self, size: int):
        lib = load()
        self._free = lib.pcbz_host_free   # bound now: __del__ may run at interpreter exit
        self.addr = lib.pcbz_host_alloc(size)
        self.size = size

    def __del__(self):
        if self.addr:
            self._free(self.addr)
            self.addr = None


class _PinnedCache(threading.local):
    """Grow-only page-locked buffer per thread (pcbz_host_alloc): device->host
    payload copies land in it at PCIe speed.  The contents are valid until
    the same thread asks for a buffer again; the memory itself stays alive
    as long as an array handed out views it (each array keeps its block)."""

    def __init__(self):
        self.block = None

    def get(self, nbytes: int) -> np.ndarray:
        if nbytes > PINNED_MAX:   # do not pin very large buffers: pageable, not cached
            return np.empty(max(int(nbytes), 1), np.uint8)
        if self.block is None or nbytes > self.block.size:
            self.block = None     # the old block lives on in the arrays still viewing it
            blk = _PinnedBlock(max(int(nbytes), 1 << 20))
            if not blk.addr:      # page-locked memory exhausted: pageable for this call
                return np.empty(max(int(nbytes), 1), np.uint8)
            self.block = blk
        buf = (ctypes.c_uint8 * self.block.size).from_address(self.block.addr)
        buf._pcbz_owner = self.block   # ndarray.base -> buf -> block
        return np.ctypeslib.as_array(buf)[:nbytes]


#: largest page-locked buffer the cache keeps per thread (bigger requests get pageable memory)
PINNED_MAX = 2 << 30

_pinned = _PinnedCache()


def pinned_buffer(nbytes: int) -> np.ndarray:
    """This thread's cached page-locked uint8 buffer of at least nbytes."""
    return _pinned.get(nbytes)


_PyBytes_FromStringAndSize = ctypes.pythonapi.PyBytes_FromStringAndSize
_PyBytes_FromStringAndSize.restype = ctypes.py_object
_PyBytes_FromStringAndSize.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
_PyBytes_AsString = ctypes.pythonapi.PyBytes_AsString
_PyBytes_AsString.restype = ctypes.c_void_p
_PyBytes_AsString.argtypes = [ctypes.py_object]


def _address(part) -> int:
    if isinstance(part, bytes):
        return _PyBytes_AsString(part)
    return np.frombuffer(part, np.uint8).ctypes.data


def join(parts, threads: int | None = None) -> bytes:
    """b"".join(parts) for bytes-like parts, the copy done by pcbz_gather on
    up to `threads` host threads into a fresh bytes object (filled before it
    is shared, the CPython PyBytes_FromStringAndSize(NULL, n) idiom)."""
    import os
    parts = [p for p in parts if len(p)]
    total = sum(len(p) for p in parts)
    out = _PyBytes_FromStringAndSize(None, total)
    n = len(parts)
    if n:
        srcs = (ctypes.c_void_p * n)(*[_address(p) for p in parts])
        lens = np.array([len(p) for p in parts], np.int64)
        check(load().pcbz_gather(_PyBytes_AsString(out), srcs, lens.ctypes.data, n,
                                 threads or (os.cpu_count() or 1)))
    return out


def copy_into(dst: np.ndarray, src) -> None:
    """dst[...] = src bytes, copied by pcbz_gather on all host threads (a
    fresh destination is first-touched in parallel)."""
    import os
    n = dst.nbytes
    srcs = (ctypes.c_void_p * 1)(_address(src))
    lens = np.array([n], np.int64)
    check(load().pcbz_gather(dst.ctypes.data, srcs, lens.ctypes.data, 1, os.cpu_count() or 1))
