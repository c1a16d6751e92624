"""TEST INFRASTRUCTURE ONLY -- the checker, never the product.

CPU restatement of the reference's entropy-judgement path
(/root/reference/pkg/src/pcbz): ctypes wrappers over oracle/pcbz_oracle.c
plus numpy/Python restatements of the host-side steps.  Only tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline leg, --impl reference)
may import this module.

Pinning: tests/test_oracle_golden.py checks every function here against
fixtures generated from the real reference (tests/golden/make_golden.py).
"""
from __future__ import annotations

import bz2
import ctypes
import struct
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboracle.so"

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        lib = ctypes.CDLL(str(LIB))
        sigs = {
            "oracle_residual_image": [_vp, _i64, _i64, ctypes.c_int, _i64, _i64, _vp],
            "oracle_reconstruct_image": [_vp, _i64, _i64, ctypes.c_int, _i64, _i64, _vp],
            "oracle_temporal_delta": [_vp, _vp, _i64, _vp],
            "oracle_temporal_undelta": [_vp, _vp, _i64, _vp],
            "oracle_counting_bwt": [_vp, _i64, _vp],
            "oracle_pair_hist": [_vp, _i64, _vp],
            "oracle_bwt_pair_hist": [_vp, _i64, _vp],
            "oracle_residual_bwt_pair_hist": [_vp, _i64, _i64, ctypes.c_int, _i64, _i64, _vp],
            "oracle_select_batch": [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, ctypes.c_int,
                                    ctypes.c_int, _vp, _vp, _vp],
        }
        for name, args in sigs.items():
            getattr(lib, name).argtypes = args
            getattr(lib, name).restype = ctypes.c_int if name == "oracle_select_batch" else None
        lib.oracle_entropy2d.argtypes = [_vp, _i64]
        lib.oracle_entropy2d.restype = ctypes.c_double
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _u16(img):
    return np.ascontiguousarray(img, dtype=np.uint16)


# ---- _kernels.py restatements ------------------------------------------------

def residual_image(img, intra_id, px, py):            # _kernels.py:46-66
    a = _u16(img)
    out = np.empty_like(a)
    load().oracle_residual_image(_p(a), a.shape[0], a.shape[1], int(intra_id), int(px), int(py), _p(out))
    return out


def reconstruct_image(res, intra_id, px, py):         # _kernels.py:69-90
    a = _u16(res)
    out = np.empty_like(a)
    load().oracle_reconstruct_image(_p(a), a.shape[0], a.shape[1], int(intra_id), int(px), int(py), _p(out))
    return out


def residual_bwt_pair_hist(img, intra_id, px, py):    # _kernels.py:157-204
    a = _u16(img)
    out = np.zeros(65536, np.int64)
    load().oracle_residual_bwt_pair_hist(_p(a), a.shape[0], a.shape[1], int(intra_id), int(px), int(py), _p(out))
    return out


def counting_bwt(s):                                  # _kernels.py:93-113
    a = np.ascontiguousarray(s, dtype=np.uint8)
    out = np.empty_like(a)
    if a.size:
        load().oracle_counting_bwt(_p(a), a.size, _p(out))
    return out


def pair_hist(s):                                     # _kernels.py:116-122
    a = np.ascontiguousarray(s, dtype=np.uint8)
    out = np.zeros(65536, np.int64)
    load().oracle_pair_hist(_p(a) if a.size else None, a.size, _p(out))
    return out


def bwt_pair_hist(s):                                 # _kernels.py:136-154
    a = np.ascontiguousarray(s, dtype=np.uint8)
    out = np.zeros(65536, np.int64)
    load().oracle_bwt_pair_hist(_p(a) if a.size else None, a.size, _p(out))
    return out


def temporal_delta(cur, prev):                        # predictors.py:116-120
    c, p = _u16(cur), _u16(prev)
    out = np.empty_like(c)
    load().oracle_temporal_delta(_p(c), _p(p), c.size, _p(out))
    return out


def temporal_undelta(delta, prev):                    # predictors.py:123-127
    d, p = _u16(delta), _u16(prev)
    out = np.empty_like(d)
    load().oracle_temporal_undelta(_p(d), _p(p), d.size, _p(out))
    return out


# ---- criterion.py / core.py restatements ---------------------------------------

def entropy2d(counts, total):                         # criterion.py:86-96 (numpy, same ops)
    if total <= 0:
        return 0.0
    c = np.asarray(counts)
    c = c[c > 0]
    p = c / float(total)
    return float(-(p * np.log2(p)).sum())


def pack_symbols(samples):                            # core.py:228-237
    return np.asarray(samples, dtype=np.uint16).astype(">u2").tobytes()


def select_predictor(frame, prev, spec_bytes, px, py):
    """criterion.py:136-173 restated: returns ([(byte, entropy)], selected byte,
    [hist]) with spec bytes sorted ascending."""
    frame = _u16(frame)
    codes = sorted(int(b) for b in spec_bytes)
    delta = temporal_delta(frame, prev) if any(b & 0x80 for b in codes) else None
    entries, hists = [], []
    for b in codes:
        img = delta if b & 0x80 else frame
        h = residual_bwt_pair_hist(img, b & 0x7F, px, py)
        hists.append(h)
        entries.append((b, entropy2d(h, 2 * img.size - 1)))
    best = min(range(len(codes)), key=lambda i: (entries[i][1], codes[i]))
    return entries, codes[best], hists


def emit_stream(frame, prev, spec_byte, px, py):
    """pack_symbols(apply_predictor(...)) -- pipeline.py:100-101."""
    src = temporal_delta(frame, prev) if spec_byte & 0x80 else _u16(frame)
    return pack_symbols(residual_image(src, spec_byte & 0x7F, px, py))


def select_batch(frames, prevs, spec_bytes, px, py, nthreads, want_stream=True):
    """Batched C restatement used for CPU-baseline timing: frames [F,H,W],
    prevs [F,H,W] or None (prev of frame f), every spec scored on every frame."""
    fr = np.ascontiguousarray(frames, dtype=np.uint16)
    F, H, W = fr.shape
    pv = None if prevs is None else np.ascontiguousarray(prevs, dtype=np.uint16)
    codes = np.array(sorted(int(b) for b in spec_bytes), np.uint8)
    ent = np.zeros((F, codes.size), np.float64)
    sel = np.zeros(F, np.uint8)
    stream = np.zeros((F, 2 * H * W), np.uint8) if want_stream else None
    load().oracle_select_batch(_p(fr), _p(pv), F, H, W, int(px), int(py), _p(codes), codes.size,
                               int(nthreads), _p(ent), _p(sel), _p(stream))
    return ent, sel, stream


# ---- pipeline / blocks / container restatements (pipeline.py, blocks.py, container.py)

def compress_blocks(stream, block_size=4 * 1024 * 1024):   # blocks.py:73-81
    n = -(-len(stream) // block_size) if len(stream) else 0
    return [bz2.compress(stream[i * block_size:(i + 1) * block_size], 9) for i in range(n)]


def write_container(width, height, px, py, block_size, frames):  # container.py:84-106
    flags = 1 if any(b & 0x80 for b, _ in frames) else 0
    out = bytearray(struct.pack("<4sBBBBIIIHHI", b"PCBZ", 1, flags, 16, 0, width, height,
                                len(frames), px, py, block_size))
    for b, blocks in frames:
        out += struct.pack("<B3xI", b, len(blocks))
        out += struct.pack(f"<{len(blocks)}Q", *(len(p) for p in blocks))
    for _, blocks in frames:
        for p in blocks:
            out += p
    return bytes(out)


def compress_stack(frames, px, py, temporal=True, candidates=None, forced=None,
                   block_size=4 * 1024 * 1024):
    """pipeline.py:76-113 restated over a [F,H,W] array; returns (container, selected bytes)."""
    frames = np.asarray(frames, dtype=np.uint16)
    intra = list(range(13))
    encoded, chosen = [], []
    prev = None
    for f in frames:
        have_prev = prev is not None and temporal
        if forced is not None:
            b = forced if have_prev else forced & 0x7F
        else:
            if candidates is None:
                cands = intra + ([0x80 | i for i in intra] if have_prev else [])
            else:
                cands = [c for c in candidates if have_prev or not c & 0x80]
            _, b, _ = select_predictor(f, prev if have_prev else None, cands, px, py)
        encoded.append((b, compress_blocks(emit_stream(f, prev, b, px, py), block_size)))
        chosen.append(b)
        prev = f
    H, W = frames.shape[1:]
    return write_container(W, H, px, py, block_size, encoded), chosen


def decompress_stack(data):
    """pipeline.py:121-139 restated (losslessness oracle): returns [F,H,W]."""
    hdr = struct.unpack_from("<4sBBBBIIIHHI", data, 0)
    width, height, nf, px, py = hdr[5], hdr[6], hdr[7], hdr[8], hdr[9]
    off = 28
    recs = []
    for _ in range(nf):
        b, nb = struct.unpack_from("<B3xI", data, off)
        off += 8
        sizes = struct.unpack_from(f"<{nb}Q", data, off)
        off += 8 * nb
        recs.append((b, sizes))
    frames, prev = [], None
    for b, sizes in recs:
        stream = b"".join(bz2.decompress(data[off + sum(sizes[:i]):off + sum(sizes[:i + 1])])
                          for i in range(len(sizes)))
        off += sum(sizes)
        res = np.frombuffer(stream, ">u2").reshape(height, width).astype(np.uint16)
        img = reconstruct_image(res, b & 0x7F, px, py)
        if b & 0x80:
            img = temporal_undelta(img, prev)
        frames.append(img)
        prev = img
    return np.stack(frames)
