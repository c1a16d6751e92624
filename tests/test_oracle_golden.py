"""Pin the CPU oracle (oracle/) against fixtures produced by the REAL reference
(tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

import oracle
from conftest import golden_hist, sha


def test_approx_bwt_kats(golden_kats):
    for s_hex, want_hex in golden_kats["approx_bwt"]:
        s = np.frombuffer(bytes.fromhex(s_hex), np.uint8)
        assert oracle.counting_bwt(s).tobytes().hex() == want_hex


def test_pair_hist_kats(golden_kats):
    for s_hex, total, bins, counts in golden_kats["pair_hist"]:
        s = np.frombuffer(bytes.fromhex(s_hex), np.uint8)
        h = oracle.pair_hist(s)
        assert int(h.sum()) == total
        assert np.nonzero(h)[0].tolist() == bins
        assert h[bins].tolist() == counts


def test_entropy_kats(golden_kats):
    for items, want_hex in golden_kats["entropy"]:
        c = np.zeros(65536, np.int64)
        for b, v in items:
            c[b] = v
        assert oracle.entropy2d(c, int(c.sum())) == float.fromhex(want_hex)


def test_residual_const7(golden_kats):
    img = np.full((2, 3), 7, np.uint16)
    assert oracle.residual_image(img, 1, 1, 1).tolist() == golden_kats["residual_const7_id1"]


def test_fused_equals_composed_random():
    rng = np.random.default_rng(5)
    for _ in range(40):
        h, w = rng.integers(1, 12, 2)
        img = rng.integers(0, 65536, (h, w), dtype=np.uint16)
        s = np.frombuffer(oracle.pack_symbols(img), np.uint8)
        assert np.array_equal(oracle.residual_bwt_pair_hist(img, 0, 1, 1),
                              oracle.pair_hist(oracle.counting_bwt(s)))
        assert np.array_equal(oracle.bwt_pair_hist(s), oracle.pair_hist(oracle.counting_bwt(s)))


def test_small_cases_histograms_entropies_streams(golden_small):
    meta, arrays = golden_small
    for name, m in meta.items():
        vol = arrays[f"{name}/frames"]
        px, py = m["px"], m["py"]
        prev = None
        for fi, fm in enumerate(m["frames"]):
            entries, selected, hists = oracle.select_predictor(vol[fi], prev, fm["codes"], px, py)
            for (code, e), h, want_e in zip(entries, hists, fm["entropies"]):
                assert np.array_equal(h, golden_hist(arrays, name, fi, code)), (name, fi, code)
                assert e == pytest.approx(float.fromhex(want_e), rel=1e-13, abs=1e-15)
            assert selected == fm["selected"], (name, fi)
            for code, want in fm["streams"].items():
                assert sha(oracle.emit_stream(vol[fi], prev, int(code), px, py)) == want
            prev = vol[fi]


def test_small_cases_containers(golden_small):
    meta, arrays = golden_small
    for name, m in meta.items():
        vol = arrays[f"{name}/frames"]
        for label, kw in [("auto", {}), ("intra", {"temporal": False}),
                          ("forced_t5", {"forced": 0x85}),
                          ("cands", {"candidates": [0x03, 0x8B, 0x0C]})]:
            data, chosen = oracle.compress_stack(vol, m["px"], m["py"], **kw)
            want = m["containers"][label]
            assert chosen == want["specs"], (name, label)
            assert len(data) == want["len"] and sha(data) == want["sha"], (name, label)
        assert np.array_equal(oracle.decompress_stack(data), vol)


@pytest.mark.slow
def test_medium_cases(golden_medium):
    from workloads.lfm_synth import SynthParams, generate_array
    for case in golden_medium:
        p = case["params"]
        vol = generate_array(SynthParams(**p))
        assert sha(vol) == case["volume_sha"]
        prev = None
        for fi, fm in enumerate(case["frames"]):
            entries, selected, hists = oracle.select_predictor(vol[fi], prev, fm["codes"],
                                                               p["pitch_x"], p["pitch_y"])
            assert [sha(h) for h in hists] == fm["hist_sha"]
            for (_, e), want in zip(entries, fm["entropies"]):
                assert e == pytest.approx(float.fromhex(want), rel=1e-13)
            assert selected == fm["selected"]
            prev = vol[fi]
        data, _ = oracle.compress_stack(vol, p["pitch_x"], p["pitch_y"])
        assert sha(data) == case["container_sha"]


@pytest.mark.slow
def test_c1_full_size_histograms(golden_c1):
    from workloads.lfm_synth import SynthParams, generate_array
    vol = generate_array(SynthParams(**golden_c1["params"]))
    entries, selected, hists = oracle.select_predictor(vol[0], None, list(range(13)), 15, 15)
    assert [sha(h) for h in hists] == golden_c1["hist_sha"]
    assert selected == golden_c1["selected"]
    for (_, e), want in zip(entries, golden_c1["entropies"]):
        assert e == pytest.approx(float.fromhex(want), rel=1e-13)
    assert sha(oracle.emit_stream(vol[0], None, selected, 15, 15)) == golden_c1["stream_sha"]


def test_select_batch_matches_python_restatement():
    rng = np.random.default_rng(3)
    vol = rng.integers(0, 4096, (3, 21, 17), dtype=np.uint16)
    prevs = np.concatenate([vol[:1], vol[:-1]])
    codes = list(range(13)) + [0x80 | i for i in range(13)]
    ent, sel, stream = oracle.select_batch(vol, prevs, codes, 4, 3, nthreads=4)
    for f in range(3):
        entries, best, _ = oracle.select_predictor(vol[f], prevs[f], codes, 4, 3)
        assert np.allclose(ent[f], [e for _, e in entries], rtol=1e-13, atol=0)
        assert sel[f] == best
        assert stream[f].tobytes() == oracle.emit_stream(vol[f], prevs[f], best, 4, 3)
