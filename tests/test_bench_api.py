"""The staged-benchmark API of the package (paper_2603_22496_b200.bench)
against the reference's own outputs (tests/golden/bench.npz, made by
tests/golden/make_bench_golden.py from kkbeam/bench.py): the seeded noise
volume bit for bit, the CSV and the console table character for character.
CPU only (no kernels)."""

import hashlib

import numpy as np

import paper_2603_22496_b200 as kb
from conftest import golden


def _rows():
    return [kb.StageTimings("kk_m5", "kk", 5, 16 / 5, 1234, 1.25, 2.5, 0.125, 3.0),
            kb.StageTimings("das", "das", 16, 1.0, 98765, 10.0, 0.5, 7.75, 20.0)]


def test_noise_volume_matches_reference():
    g = golden("bench")
    arr = kb.TransducerArray(16, 0.3e-3, 5.0e6, 20.0e6, 0.6)
    par = kb.AcquisitionParams(1540.0, np.array([-0.1, 0.0, 0.1]), 256)
    vol = kb.noise_volume(arr, par, seed=7)
    assert tuple(vol.data.shape) == tuple(g["volume_shape"])
    assert hashlib.sha256(vol.data.tobytes()).hexdigest() == str(g["volume_sha"])


def test_csv_and_table_match_reference():
    g = golden("bench")
    assert kb.bench_csv_text(_rows()) == str(g["csv"])
    assert kb.format_bench_table(_rows()) == str(g["table"])


def test_stage_timings_fields():
    r = _rows()[0]
    assert kb.STAGES == ("reorg_fft", "hilbert_compress", "ifft", "beamform")
    assert r.total_ms == 1.25 + 2.5 + 0.125 + 3.0
    assert [r.stage_ms(s) for s in kb.STAGES] == [1.25, 2.5, 0.125, 3.0]
