"""KKRF container (rffile.py mirror) against files written by the reference.

Host-side I/O through libkkb's native reader/writer (no GPU needed): the
goldens under tests/golden/kkrf were written by the reference's
write_container, and kkrf.npz holds what its read_container returned and the
FileFormatError text it raised for each corruption (make_kkrf_golden.py).
"""

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
from make_kkrf_golden import CORRUPTIONS, corrupt  # noqa: E402

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import rffile  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
G = np.load(os.path.join(GOLD, "kkrf.npz"))
NAMES = ["real", "analytic", "compressed"]


def _path(name):
    return os.path.join(GOLD, "kkrf", f"{name}.kkrf")


@pytest.mark.parametrize("name", NAMES)
def test_read_matches_reference(name):
    c = rffile.read_container(_path(name))
    assert type(c).__name__ == {"real": "RFVolume", "analytic": "AnalyticRF",
                                "compressed": "CompressedRF"}[name]
    assert c.data.dtype == G[f"{name}_data"].dtype
    assert np.array_equal(c.data, G[f"{name}_data"])
    assert np.array_equal(c.params.transmit_angles, G[f"{name}_tx"])
    meta = G[f"{name}_meta"]
    assert (c.params.sound_speed, c.params.start_time, c.params.num_samples) == \
        (meta[0], meta[1], int(meta[2]))
    if name == "compressed":
        assert c.array is None
        assert np.array_equal(c.receive_angles.angles, G["compressed_rx"])
        assert c.sampling_frequency == float(G["compressed_fs"])
    else:
        a = c.array
        assert np.array_equal([a.num_elements, a.pitch, a.center_frequency, a.sampling_frequency,
                               a.fractional_bandwidth], G[f"{name}_array"])


@pytest.mark.parametrize("name", NAMES)
def test_write_is_byte_identical(name, tmp_path):
    c = rffile.read_container(_path(name))
    out = tmp_path / "w.kkrf"
    rffile.write_container(str(out), c)
    assert out.read_bytes() == open(_path(name), "rb").read()


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("label,off,rep", CORRUPTIONS, ids=[c[0] for c in CORRUPTIONS])
def test_corruptions_raise_like_reference(name, label, off, rep, tmp_path):
    key = f"{name}_err_{label}"
    if key not in G.files:
        pytest.skip("not applicable to this kind")
    bad = tmp_path / "bad.kkrf"
    bad.write_bytes(corrupt(open(_path(name), "rb").read(), off, rep))
    want = str(G[key])
    if want == "OK":
        rffile.read_container(str(bad))
        return
    with pytest.raises(kb.DataError) as ei:
        rffile.read_container(str(bad))
    got = f"{type(ei.value).__name__}: {ei.value}".replace(str(bad), "<path>")
    assert got == want


def test_unserializable_and_missing_file(tmp_path):
    with pytest.raises(kb.FileFormatError, match="cannot serialize dict"):
        rffile.write_container(str(tmp_path / "x.kkrf"), {})
    with pytest.raises(OSError):
        rffile.read_container(str(tmp_path / "missing.kkrf"))
