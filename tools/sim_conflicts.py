"""Offline analysis of the judge's shared-atomic pattern on real inputs:
bin distribution, hot-bin share and simulated bank conflicts per warp ATOMS
(32 lanes = 32 runs at the same event slot).  CPU only (uses the oracle)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
import oracle  # noqa: E402
from workloads.lfm_synth import SynthParams, generate_array  # noqa: E402


def events(res):
    r = res.astype(np.int64).ravel()
    hi, lo = r >> 8, r & 0xFF
    key = np.empty(2 * r.size, np.int64); prd = np.empty_like(key)
    key[0::2], key[1::2] = hi, lo
    prd[1::2] = hi
    prd[0::2] = np.concatenate([[lo[-1]], lo[:-1]])
    return key, prd


def lane_bins(key, prd, nlanes=192):
    n = key.size
    bounds = (np.arange(nlanes + 1) * (n // 16) // nlanes) * 16   # chunk aligned (16 events/chunk)
    lane = np.searchsorted(bounds, np.arange(n), side="right") - 1
    # previous event with the same key inside the same lane
    order = np.lexsort((np.arange(n), key, lane))
    k_s, l_s = key[order], lane[order]
    same = np.zeros(n, bool); same[1:] = (k_s[1:] == k_s[:-1]) & (l_s[1:] == l_s[:-1])
    last = np.full(n, -1, np.int64)
    last_sorted = np.full(n, -1, np.int64); last_sorted[1:] = prd[order][:-1]
    last[order] = np.where(same, last_sorted, -1)
    return last, lane, bounds


def analyse(img, cid, px=15, py=15):
    res = oracle.residual_image(img, cid, px, py)
    key, prd = events(res)
    last, lane, bounds = lane_bins(key, prd)
    seen = last >= 0
    bins = np.where(seen, last * 256 + prd, -1)
    hot = seen & np.isin(bins, [0x0000, 0x00FF, 0xFF00, 0xFFFF])
    word = np.where(seen, bins >> 1, 32768 + (prd >> 1))
    bank = word % 32
    # warp w, slot s: lanes 32w..32w+31, each at its own event index bounds[l] + s
    per_lane = (bounds[1:] - bounds[:-1]).min()
    steps = min(per_lane, 4096)
    wf_tot, cnt = 0, 0
    wf_nohot = 0
    for w in range(6):
        ls = np.arange(32 * w, 32 * w + 32)
        idx = bounds[ls][:, None] + np.arange(steps)[None, :]       # [32, steps]
        b = bank[idx]; hv = hot[idx]
        for s in range(0, steps, 7):
            col = b[:, s]
            wf_tot += np.bincount(col, minlength=32).max(); cnt += 1
            cold = col[~hv[:, s]]
            wf_nohot += np.bincount(cold, minlength=32).max() if cold.size else 0
    ev_b = np.arange(key.size) % 2 == 1
    return dict(cid=cid, hot=hot.mean(), hot_B=hot[ev_b].mean(), hot_A=hot[~ev_b].mean(),
                wavefronts=wf_tot / cnt, wavefronts_without_hot=wf_nohot / cnt,
                distinct_bins=np.unique(bins[seen]).size)


if __name__ == "__main__":
    for amp, sig, ph, seed in [(20000.0, 0.0, 0.05, 1), (3000.0, 100.0, 0.05, 40), (3000.0, 500.0, 0.01, 80)]:
        img = generate_array(SynthParams(2048, 2048, 15, 15, mode="beads", signal_amplitude=amp,
                                         noise_sigma=sig, photon_scale=ph, seed=seed))[0][:512]
        print(f"beads amp={amp} sigma={sig}")
        for cid in (0, 1, 4, 7, 11):
            d = analyse(img, cid)
            print("   ", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items()})


def swizzle_study(img, cid, px=15, py=15):
    res = oracle.residual_image(img, cid, px, py)
    key, prd = events(res)
    last, lane, bounds = lane_bins(key, prd)
    seen = last >= 0
    L = np.where(seen, last, 0x100)
    word = L * 128 + (prd >> 1)
    fns = {
        "none": lambda w, L, p: w % 32,
        "xor_last": lambda w, L, p: ((p >> 1) ^ L) % 32,
        "xor_last_rot": lambda w, L, p: ((p >> 1) ^ (L >> 3) ^ (L << 2)) % 32,
        "add_mul": lambda w, L, p: ((p >> 1) + L * 13) % 32,
        "xor_last_hi": lambda w, L, p: ((p >> 1) ^ L ^ (L >> 5)) % 32,
    }
    out = {}
    per_lane = (bounds[1:] - bounds[:-1]).min()
    steps = min(per_lane, 4096)
    for name, fn in fns.items():
        bank = fn(word, L, prd)
        tot = cnt = 0
        for w in range(6):
            ls = np.arange(32 * w, 32 * w + 32)
            idx = bounds[ls][:, None] + np.arange(0, steps, 7)[None, :]
            b = bank[idx]
            for s in range(b.shape[1]):
                tot += np.bincount(b[:, s], minlength=32).max(); cnt += 1
        out[name] = round(tot / cnt, 2)
    return out
