"""Benchmark / test workloads (harness input, not product code): the
reference's synthetic light-field generator restated bit-for-bit
(lfm_synth.py, pinned by tests/golden/synth_hashes.json) and the BASELINE
configurations C1-C4 built from it (configs.py)."""
