"""KKRF payloads streamed to / from HBM (pinned double-buffered staging)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import _device as dev  # noqa: E402
from paper_2603_22496_b200 import rffile  # noqa: E402


def _volume(seed, T=20011):
    # 2 x 128 x 20011 float32 = 20.5 MB: two 16 MiB staging chunks, ragged tail
    arr = kb.TransducerArray(128, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    p = kb.AcquisitionParams(1540.0, kb.transmit_angles(2, np.deg2rad(5)), T, start_time=2e-6)
    data = np.random.default_rng(seed).standard_normal((2, 128, T)).astype(np.float32)
    return kb.RFVolume(data, arr, p)


def test_device_read_write_roundtrip(tmp_path):
    v = _volume(0)
    path = str(tmp_path / "v.kkrf")
    rffile.write_container(path, v)
    d = rffile.read_container_device(path)
    assert d.kind == rffile.KIND_REAL and tuple(d.data.shape) == v.data.shape
    assert np.array_equal(dev.to_host(d.data), v.data)
    assert d.array.num_elements == 128 and d.params.num_samples == 20011
    out = str(tmp_path / "w.kkrf")
    rffile.write_container_device(out, d, d.data)
    assert open(out, "rb").read() == open(path, "rb").read()


@pytest.mark.parametrize("threads", [None, 1, 2, 5])
def test_ensemble_into_one_tensor(tmp_path, threads):
    # several reader threads (kkb_kkrf_read_ensemble); frames larger than one
    # 16 MiB staging chunk (T = 20011) exercise the double buffering per thread
    paths = []
    frames = []
    for f in range(5):
        v = _volume(f, T=2048)
        paths.append(str(tmp_path / f"f{f}.kkrf"))
        rffile.write_container(paths[-1], v)
        frames.append(v.data)
    t, meta = rffile.read_ensemble_device(paths, threads=threads)
    assert tuple(t.shape) == (5, 2, 128, 2048)
    assert np.array_equal(dev.to_host(t), np.stack(frames))
    big = []
    for f in range(3):
        v = _volume(10 + f, T=20011)
        big.append(str(tmp_path / f"b{f}.kkrf"))
        rffile.write_container(big[-1], v)
        frames.append(v.data)
    tb, _ = rffile.read_ensemble_device(big, threads=threads)
    assert np.array_equal(dev.to_host(tb), np.stack(frames[5:]))
    other = _volume(9, T=1024)
    rffile.write_container(str(tmp_path / "odd.kkrf"), other)
    with pytest.raises(kb.FileFormatError, match="geometry differs"):
        rffile.read_ensemble_device(paths + [str(tmp_path / "odd.kkrf")])


def test_compressed_device_roundtrip(tmp_path):
    rx = kb.explicit_angles(np.deg2rad([-1.0, 0.0, 1.0]), np.deg2rad(5))
    p = kb.AcquisitionParams(1540.0, kb.transmit_angles(2, np.deg2rad(5)), 64)
    z = np.random.default_rng(4).standard_normal((2, 3, 64, 2)).view(np.complex128)[..., 0]
    c = kb.CompressedRF(z.astype(np.complex64), rx, p, sampling_frequency=20.8e6)
    path = str(tmp_path / "c.kkrf")
    rffile.write_container(path, c)
    d = rffile.read_container_device(path)
    assert np.array_equal(dev.to_host(d.data), c.data)
    assert np.array_equal(d.receive_angles.angles, rx.angles)
