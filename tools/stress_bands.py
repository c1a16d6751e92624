"""Randomised parity stress of the band-sharded judge: random
frame shapes, pitches, value kinds, band counts, halo / no halo, band views
whose rows outside the band are garbage, owner-computes (collective or
peer-memory exchange) or replicated merge.
Every case must equal the whole-frame device judge bit for bit (entropies,
selections, concatenated band streams) and, for the selections and streams,
the oracle.  Runs on one GPU with the rank exchange emulated
(shard.emulate_band_exchange, through tests/test_gpu_parity._run_bands).

    python tools/stress_bands.py [cases] [seed]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle"), str(ROOT / "tests")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (the checker)
from stress_parity import frame, tie_note  # noqa: E402
from test_gpu_parity import _run_bands  # noqa: E402
from paper_2310_09467_b200.device import DeviceJudge  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--only=")]
    only = {int(x) for a in sys.argv[1:] if a.startswith("--only=") for x in a[7:].split(",")}
    cases = int(args[0]) if len(args) > 0 else 100
    rng = np.random.default_rng(int(args[1]) if len(args) > 1 else 11)
    codes = list(range(13)) + [0x80 | i for i in range(13)]
    bad = 0
    for t in range(cases):
        F = int(rng.integers(1, 4))
        H = int(rng.integers(8, 260))
        W = int(rng.integers(8, 400))
        px, py = int(rng.integers(1, 20)), int(rng.integers(1, 31))
        nb = int(rng.integers(1, 9))
        halo = bool(rng.integers(0, 2))
        rows_only = bool(rng.integers(0, 2))
        merge = int(rng.integers(0, 4))          # 0 replicated, 1 owner-computes (NCCL form), 2-3 peer
        replicated, peer = merge == 0, merge >= 2
        kind = str(rng.choice(["smooth", "full", "narrow", "const"]))
        vol = np.stack([frame(rng, H, W, kind) for _ in range(F + 1)])
        if only and t not in only:
            continue
        frames = torch.from_numpy(np.ascontiguousarray(vol[1:] if halo else vol[:F])).cuda()
        halo_t = torch.from_numpy(np.ascontiguousarray(vol[0])).cuda() if halo else None
        whole = DeviceJudge((F, H, W), (px, py), codes, temporal=True)
        e0, s0, st0 = (x.cpu().numpy() for x in whole(frames, halo_t))
        ent, sel, streams = _run_bands(frames, halo_t, (F, H, W), (px, py), codes, True, nb,
                                       rows_only, replicated, peer)
        why = []
        if not np.array_equal(ent, e0, equal_nan=True):
            d = np.argwhere(~((ent == e0) | (np.isnan(ent) & np.isnan(e0))))
            why.append(f"entropies differ from the whole-frame judge at {d[:4].tolist()} "
                       f"({[(ent[tuple(i)], e0[tuple(i)]) for i in d[:2]]})")
        if not np.array_equal(sel, s0):
            why.append(f"selections {sel.tolist()} vs whole {s0.tolist()}")
        if not np.array_equal(streams, st0):
            why.append(f"streams differ from the whole-frame judge in frames "
                       f"{sorted(set(np.argwhere(streams != st0)[:, 0].tolist()))}")
        # the oracle on the selections and streams
        fr = vol[1:] if halo else vol[:F]
        p = vol[0] if halo else None
        for f in range(F):
            cands = codes if p is not None else list(range(13))
            _, best, hh = oracle.select_predictor(fr[f], p, cands, px, py)
            if int(sel[f]) != best:
                why.append(f"frame {f} selection {int(sel[f]):#x} vs oracle {best:#x}: "
                           + tie_note(hh, cands, int(sel[f]), best))
            if streams[f].tobytes() != oracle.emit_stream(fr[f], p, int(sel[f]), px, py):
                why.append(f"frame {f} stream vs oracle")
            p = fr[f]
        if why:
            bad += 1
            print(f"MISMATCH case {t}: F={F} {H}x{W} pitch {px}x{py} {kind} bands {nb} halo {halo} "
                  f"rows_only {rows_only} merge {('replicated', 'owner', 'peer', 'peer')[merge]}: " + "; ".join(why), flush=True)
    print(f"{cases} band cases, {bad} mismatches", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
