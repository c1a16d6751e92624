"""Compress / decompress round trip on a bench workload (default: the C3
100-frame series, temporal on): whole-pipeline wall times with bzip2 on all
host threads, losslessness, and the device inverse-prediction step
(pcbz_reconstruct_host: H2D of residuals, reconstruct + undelta kernels,
D2H) timed on its own.

    python tools/roundtrip.py [workload] [nframes]
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2310_09467_b200 import (CompressOptions, Frame, FrameStack, LensletGeometry, _lib,  # noqa: E402
                                   compress_stack_detailed, decompress_stack, read_container)
from paper_2310_09467_b200.codec import decompress_blocks, CompressedBlocks, BlockPlan  # noqa: E402
from paper_2310_09467_b200.core import unpack_symbols  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    wl = bench.WORKLOADS[name]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else wl.frames
    cores = os.cpu_count() or 1
    vol = bench.make_frames(wl, range(n), cores)
    geo = LensletGeometry(wl.pitch, wl.pitch)
    stack = FrameStack(tuple(Frame(f, geo) for f in vol))
    opts = CompressOptions(workers=cores, temporal=wl.temporal,
                           candidates=None if wl.temporal else tuple(
                               __import__("paper_2310_09467_b200").all_intra_specs()))
    compress_stack_detailed(stack, opts)   # warm-up at full size: context, device buffers
    t0 = time.perf_counter()
    res = compress_stack_detailed(stack, opts)
    t_c = time.perf_counter() - t0
    t0 = time.perf_counter()
    back = decompress_stack(res.data, workers=cores)
    t_d = time.perf_counter() - t0
    lossless = bool(np.array_equal(back.to_array(), vol))
    # the device inverse-prediction step alone
    header, records, payloads = read_container(res.data)
    H, W = header.height, header.width
    resid = np.empty((n, H, W), np.uint16)
    for i, rec in enumerate(records):
        blocks = CompressedBlocks(BlockPlan(header.block_size, len(rec.block_sizes)),
                                  tuple(bytes(p) for p in payloads[i]))
        resid[i] = unpack_symbols(decompress_blocks(blocks, cores), W, H)
    sel = np.array([r.spec.to_byte() for r in records], np.uint8)
    out = np.empty_like(resid)
    lib = _lib.load()
    for _ in range(2):
        t0 = time.perf_counter()
        _lib.check(lib.pcbz_reconstruct_host(_lib.ptr(resid), None, n, H, W, wl.pitch, wl.pitch,
                                             _lib.ptr(sel), _lib.ptr(out)))
        t_r = time.perf_counter() - t0
    raw = vol.nbytes
    print(json.dumps({
        "workload": wl.description, "frames": n, "raw_bytes": raw, "container_bytes": len(res.data),
        "compression_ratio": raw / len(res.data), "host_threads": cores,
        "compress_s": t_c, "compress_GBps": raw / t_c / 1e9, "device_judge_s": res.select_seconds,
        "device_encode_calls_s": res.encode_seconds, "coder": opts.coder,
        "decompress_s": t_d, "decompress_GBps": raw / t_d / 1e9, "lossless": lossless,
        "reconstruct_host_call_s": t_r, "reconstruct_GBps": raw / t_r / 1e9,
        "modes": {f"0x{c:02X}": int((sel == c).sum()) for c in np.unique(sel)}}), flush=True)


if __name__ == "__main__":
    main()
