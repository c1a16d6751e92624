"""Randomised stress of the GPU bzip2 coder and decoder against libbzip2:
random inputs (up to ~3 MB; alphabets of 2..256 symbols, run-heavy and
noisy mixes, every compression level for the decoder) -- the coder must
produce bz2.compress(x, 9) byte for byte, the decoder must return x for
every stream it takes (only exactly periodic blocks may be left to the
host).  python tools/stress_bzip2.py [cases] [seed]
"""
import bz2
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2310_09467_b200 import _lib  # noqa: E402
from paper_2310_09467_b200.codec import bz2_blocks_device  # noqa: E402


def sample(rng):
    n = int(rng.choice([1, 7, 100, 5000, 90_000, 600_000, 1_200_000, 3_000_000]))
    alph = int(rng.choice([2, 3, 16, 64, 256]))
    mode = rng.integers(0, 3)
    if mode == 0:
        return rng.integers(0, alph, n, dtype=np.uint8).tobytes()
    if mode == 1:
        vals = rng.integers(0, alph, n // 8 + 1, dtype=np.uint8)
        reps = rng.integers(1, 30, vals.size)
        return np.repeat(vals, reps)[:n].tobytes()
    return (rng.normal(128, rng.choice([1, 10, 60]), n).clip(0, 255).astype(np.uint8)).tobytes()


def device_decode(payloads, sizes):
    n = len(payloads)
    ptrs = (ctypes.c_void_p * n)(*[_lib._address(p) for p in payloads])
    lens = np.array([len(p) for p in payloads], np.int64)
    osz = np.array(sizes, np.int64)
    off = np.zeros(n, np.int64)
    off[1:] = np.cumsum(osz)[:-1]
    out = np.empty(max(int(osz.sum()), 1), np.uint8)
    st = np.ones(n, np.uint8)
    _lib.check(_lib.load().pcbz_bunzip2_host(ptrs, lens.ctypes.data, n, out.ctypes.data, off.ctypes.data,
                                             osz.ctypes.data, st.ctypes.data))
    return st, [out[off[i]:off[i] + osz[i]].tobytes() for i in range(n)]


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
    inputs = [sample(rng) for _ in range(cases)]
    levels = [int(rng.integers(1, 10)) for _ in range(cases)]
    enc_bad = sum(g != bz2.compress(x, 9) for g, x in zip(bz2_blocks_device(inputs), inputs))
    payloads = [bz2.compress(x, lv) for x, lv in zip(inputs, levels)]
    st, got = device_decode(payloads, [len(x) for x in inputs])
    dec_bad = sum(1 for s, g, x in zip(st, got, inputs) if s == 0 and g != x)
    taken = int((st == 0).sum())
    print(f"{cases} inputs ({sum(map(len, inputs)) / 1e6:.0f} MB): coder mismatches {enc_bad}, "
          f"decoder took {taken}, decoder mismatches {dec_bad}", flush=True)
    return 1 if enc_bad or dec_bad else 0


if __name__ == "__main__":
    sys.exit(main())
