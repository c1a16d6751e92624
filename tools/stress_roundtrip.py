"""Randomised end-to-end stress of the public API against the oracle:
random stacks (1-24 frames, any width, pitches up to 80 x 40, value kinds),
temporal on/off, random candidate subsets or a forced predictor, tiny to
default bzip2 block sizes, device or host bzip2 coder.  Every case must give

  * compress_stack == oracle.compress_stack, byte for byte (the reference's
    container, pipeline.py:76-113 / container.py:84-106),
  * decompress_stack(container) == the input (device bzip2 decoder where it
    takes the container, GPU inverse prediction incl. the band wavefront
    kernel for pitch_x <= 64, pitch_y <= 31),
  * the pipelined host judge (pcbz_judge_host; run as a script, in chunks of
    3 frames with a halo across chunks) == the oracle's selections and streams.

    python tools/stress_roundtrip.py [cases] [seed] [--only=i,j]
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle"), str(ROOT / "tools")]

import numpy as np  # noqa: E402

import oracle  # noqa: E402  (the checker)
from stress_parity import frame  # noqa: E402
from paper_2310_09467_b200 import (CompressOptions, Frame, FrameStack, LensletGeometry,  # noqa: E402
                                   PredictorSpec, compress_stack, decompress_stack, pipeline)

ALL = list(range(13)) + [0x80 | i for i in range(13)]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--only=")]
    only = {int(x) for a in sys.argv[1:] if a.startswith("--only=") for x in a[7:].split(",")}
    cases = int(args[0]) if len(args) > 0 else 100
    rng = np.random.default_rng(int(args[1]) if len(args) > 1 else 5)
    bad = 0
    for t in range(cases):
        F = int(rng.integers(1, 25))
        H = int(rng.integers(1, 160))
        W = int(rng.integers(1, 260))
        px, py = int(rng.integers(1, 81)), int(rng.integers(1, 41))
        kind = str(rng.choice(["smooth", "smooth", "full", "narrow", "const"]))
        vol = np.stack([frame(rng, H, W, kind) for _ in range(F)])
        temporal = bool(rng.integers(0, 4) > 0)
        mode = int(rng.integers(0, 6))          # 0-3 default set, 4 subset, 5 forced
        cands = forced = None
        if mode == 4:
            k = int(rng.integers(1, 27))
            cands = sorted(int(c) for c in rng.choice(ALL, k, replace=False))
            if not any(c < 0x80 for c in cands):
                cands = sorted(cands + [int(rng.integers(0, 13))])
        elif mode == 5:
            forced = int(rng.choice(ALL))
        block = int(rng.choice([300, 5000, 4 * 1024 * 1024]))
        coder = str(rng.choice(["device", "host"]))
        if only and t not in only:
            continue
        geo = LensletGeometry(px, py)
        opts = CompressOptions(candidates=None if cands is None else tuple(PredictorSpec.from_byte(c) for c in cands),
                               forced=None if forced is None else PredictorSpec.from_byte(forced),
                               block_size=block, workers=2, temporal=temporal, coder=coder)
        why = []
        try:
            data = compress_stack(FrameStack(tuple(Frame(f, geo) for f in vol)), opts)
            want, chosen = oracle.compress_stack(vol, px, py, temporal=temporal, candidates=cands,
                                                 forced=forced, block_size=block)
            if data != want:
                why.append("container")
            back = decompress_stack(data, workers=2)
            if not np.array_equal(np.stack([f.samples for f in back.frames]), vol):
                why.append("round trip")
            # the pipelined host judge over the default candidate set
            codes = ALL if temporal else list(range(13))
            ent, sel, streams = pipeline.judge_volume(vol, geo, codes, temporal)
            p = None
            for f in range(F):
                have_prev = p is not None
                fc = codes if have_prev else list(range(13))
                _, best, _ = oracle.select_predictor(vol[f], p, fc, px, py)
                if int(sel[f]) != best:
                    why.append(f"host judge frame {f} selection {int(sel[f]):#x} vs {best:#x}")
                elif streams[f].tobytes() != oracle.emit_stream(vol[f], p, best, px, py):
                    why.append(f"host judge frame {f} stream")
                p = vol[f] if temporal else None
        except Exception as e:  # noqa: BLE001 -- a stress case must not raise
            why.append(f"raised {type(e).__name__}: {e}")
        if why:
            bad += 1
            print(f"MISMATCH case {t}: F={F} {H}x{W} pitch {px}x{py} {kind} temporal {temporal} "
                  f"cands {cands} forced {forced} block {block} coder {coder}: " + "; ".join(why[:4]),
                  flush=True)
    print(f"{cases} round-trip cases, {bad} mismatches", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    # read once per process by the library (first pcbz_judge_host call):
    # pipeline every call, a halo across every chunk boundary
    os.environ.setdefault("PCBZ_HOST_CHUNK", "3")
    sys.exit(main())
