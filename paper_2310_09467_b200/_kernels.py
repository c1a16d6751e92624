"""Drop-in replacements for the reference's compiled kernels
(reference pkg/src/pcbz/_kernels.py), executed on the B200 through
libpcbz_b200.so.  Same names, argument meaning and return types as the
numba originals; inputs are borrowed, outputs are fresh arrays.
"""
from __future__ import annotations

import numpy as np

from . import _lib


def _img(img) -> np.ndarray:
    a = np.ascontiguousarray(img)
    if a.dtype != np.uint16 or a.ndim != 2:
        raise TypeError("expected a 2D uint16 image")
    return a


def _bytes(s) -> np.ndarray:
    a = np.ascontiguousarray(s)
    if a.dtype != np.uint8 or a.ndim != 1:
        raise TypeError("expected a 1D uint8 array")
    return a


def residual_bwt_pair_hist(img, intra_id, px, py) -> np.ndarray:
    """int64[65536] approximate-BWT pair histogram of one predictor's packed
    residual stream (reference _kernels.py:157-204)."""
    a = _img(img)
    out = np.zeros(65536, np.int64)
    h, w = a.shape
    _lib.check(_lib.load().pcbz_residual_bwt_pair_hist(_lib.ptr(a), h, w, int(intra_id), int(px),
                                                       int(py), _lib.ptr(out)))
    return out


def residual_image(img, intra_id, px, py) -> np.ndarray:
    """Symbol image of one intra predictor (reference _kernels.py:46-66)."""
    a = _img(img)
    out = np.empty_like(a)
    h, w = a.shape
    _lib.check(_lib.load().pcbz_residual_image(_lib.ptr(a), h, w, int(intra_id), int(px), int(py),
                                               _lib.ptr(out)))
    return out


def counting_bwt(s) -> np.ndarray:
    """First-byte stable rotation sort, last column (reference _kernels.py:93-113)."""
    a = _bytes(s)
    out = np.empty_like(a)
    if a.size:
        _lib.check(_lib.load().pcbz_counting_bwt(_lib.ptr(a), a.size, _lib.ptr(out)))
    return out


def pair_hist(s) -> np.ndarray:
    """Overlapping byte-pair histogram (reference _kernels.py:116-122)."""
    a = _bytes(s)
    out = np.zeros(65536, np.int64)
    _lib.check(_lib.load().pcbz_pair_hist(_lib.ptr(a) if a.size else None, a.size, _lib.ptr(out)))
    return out


def bwt_pair_hist(s) -> np.ndarray:
    """pair_hist(counting_bwt(s)) (reference _kernels.py:136-154)."""
    a = _bytes(s)
    out = np.zeros(65536, np.int64)
    _lib.check(_lib.load().pcbz_bwt_pair_hist(_lib.ptr(a) if a.size else None, a.size,
                                              _lib.ptr(out)))
    return out


def reconstruct_image(res, intra_id, px, py) -> np.ndarray:
    """Inverse of residual_image on the device (reference _kernels.py:69-90):
    the causal row-major recurrence as anti-diagonal wavefronts
    (pcbz_reconstruct_host, one frame, non-temporal mode byte)."""
    r = _img(res)
    if not 0 <= int(intra_id) <= 12:
        raise ValueError(f"intra predictor id must be in [0, 12], got {intra_id}")
    out = np.empty_like(r)
    sel = np.array([int(intra_id)], np.uint8)
    _lib.check(_lib.load().pcbz_reconstruct_host(_lib.ptr(r), None, 1, r.shape[0], r.shape[1], int(px),
                                                 int(py), _lib.ptr(sel), _lib.ptr(out)))
    return out


def temporal_delta_samples(cur: np.ndarray, prev: np.ndarray) -> np.ndarray:
    """(cur - prev) mod 2^16 on the device (reference predictors.py:116-120)."""
    c = np.ascontiguousarray(cur, dtype=np.uint16)
    p = np.ascontiguousarray(prev, dtype=np.uint16)
    out = np.empty_like(c)
    _lib.check(_lib.load().pcbz_temporal_delta(_lib.ptr(c), _lib.ptr(p), c.size, _lib.ptr(out)))
    return out


def warm_up():
    """Load the library and touch the device once (reference _kernels.py:207-216)."""
    img = np.arange(12, dtype=np.uint16).reshape(3, 4)
    residual_bwt_pair_hist(img, 3, 2, 2)
