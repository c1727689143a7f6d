"""K8 forward simulator vs the reference's RF (bit-exact).

Pins: the SHA-256 of the reference's own simulate_rf output for the config-1
point targets (with noise) and the das point dataset (tests/golden,
make_golden.py), plus the C restatement of _render_traces (oracle) on seeded
speckle with and without geometric spreading.
"""

import numpy as np
import pytest

from conftest import C, golden, sha

pytestmark = pytest.mark.gpu

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import configs  # noqa: E402


def test_config1_points_match_reference_sha():
    w = configs.config1()
    g = golden("config1")
    pulse = kb.make_pulse(5e6, 0.44, 20e6)
    assert np.array_equal(pulse.waveform, g["pulse"])
    ph = kb.Phantom(g["phantom_x"], g["phantom_z"], np.ones(5))
    rf = kb.simulate_rf(w.array, w.params, ph, pulse, noise_rms=1e-3, seed=0)
    assert rf.data.dtype == np.float32
    assert sha(rf.data) == str(g["rf_sha"])


def test_das_point_dataset_matches_reference_sha(small_array):
    g = golden("das_point")
    params = kb.AcquisitionParams(C, kb.transmit_angles(7, np.deg2rad(12)), 1024)
    ph = kb.Phantom([0.0, 1.1e-3, -0.9e-3], [9e-3, 11e-3, 12.5e-3], [1.0, 0.7, 0.9])
    rf = kb.simulate_rf(small_array, params, ph, kb.make_pulse(5.2e6, 0.67, 20.83e6))
    assert sha(rf.data) == str(g["rf_sha"])


@pytest.mark.parametrize("spread", [False, True])
def test_speckle_bit_identical_to_oracle(oracle, spread):
    arr = kb.TransducerArray(48, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    params = kb.AcquisitionParams(C, kb.transmit_angles(5, np.deg2rad(10)), 1536, start_time=2e-6)
    ph = kb.speckle_phantom((-6e-3, 6e-3, 4e-3, 22e-3), 2.0e7, seed=3,
                            inclusion_center=(0.0, 12e-3), inclusion_radius=2e-3)
    assert 3000 < len(ph) < 5000
    pulse = kb.make_pulse(5.2e6, 0.6, 20.8e6)
    rf = kb.simulate_rf(arr, params, ph, pulse, geometric_spreading=spread)
    ref = oracle.simulate_rf(arr.positions, params.transmit_angles, C, 1536, 2e-6,
                             arr.sampling_frequency, ph.x, ph.z, ph.reflectivity, pulse.waveform,
                             spread=spread)
    assert np.array_equal(rf.data, ref)


def test_echoes_clipped_before_window_and_accumulated(oracle):
    # start_time after some echoes begin: the reference clips j0 at 0; and the
    # device entry point accumulates onto a preloaded volume
    arr = kb.TransducerArray(16, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    params = kb.AcquisitionParams(C, kb.transmit_angles(3, np.deg2rad(8)), 512, start_time=6e-6)
    ph = kb.wire_phantom([1e-3, 1.5e-3, 2e-3], depth=5e-3, reflectivity=2.0)
    pulse = kb.make_pulse(5.2e6, 0.6, 20.8e6)
    ref = oracle.simulate_rf(arr.positions, params.transmit_angles, C, 512, 6e-6,
                             arr.sampling_frequency, ph.x, ph.z, ph.reflectivity, pulse.waveform)
    assert np.array_equal(kb.simulate_rf(arr, params, ph, pulse).data, ref)
    from paper_2603_22496_b200 import _device as dev

    base = np.random.default_rng(1).standard_normal((3, 16, 512)).astype(np.float32)
    out = kb.render_rf_device(arr, params, ph, pulse, out=dev.to_device(base))
    ref2 = base.copy()  # the C restatement accumulates into its output, like _render_traces
    oracle.lib().oracle_render_traces(
        oracle._ptr(ref2), 3, 16, 512, oracle._ptr(ph.x.copy()), oracle._ptr(ph.z.copy()),
        oracle._ptr(ph.reflectivity.copy()), len(ph), oracle._ptr(arr.positions),
        oracle._ptr(np.sin(params.transmit_angles)), oracle._ptr(np.cos(params.transmit_angles)),
        1.0 / C, arr.sampling_frequency, 6e-6, oracle._ptr(pulse.waveform.copy()),
        pulse.waveform.size, float(pulse.peak_index), 0, 0)
    assert np.array_equal(dev.to_host(out), ref2)


def test_window_overflow_names_the_scatterer():
    arr = kb.TransducerArray(16, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    params = kb.AcquisitionParams(C, kb.transmit_angles(3, np.deg2rad(8)), 256)
    ph = kb.Phantom([0.0, 1e-3], [3e-3, 20e-3], [1.0, 1.0])
    with pytest.raises(kb.WindowOverflowError, match=r"scatterer 1 at \(0.001, 0.02\) m needs"):
        kb.simulate_rf(arr, params, ph, kb.make_pulse(5.2e6, 0.6, 20.8e6))


def test_empty_phantom_and_noise_only():
    arr = kb.TransducerArray(8, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    params = kb.AcquisitionParams(C, [0.0], 128)
    rf = kb.simulate_rf(arr, params, kb.Phantom([], [], []), kb.make_pulse(5.2e6, 0.6, 20.8e6),
                        noise_rms=0.5, seed=7)
    ref = 0.5 * np.random.default_rng(7).standard_normal((1, 8, 128), dtype=np.float32)
    assert np.array_equal(rf.data, np.zeros((1, 8, 128), np.float32) + ref)


def test_segmented_traces_bit_identical(oracle, monkeypatch):
    # long traces are split into warp-owned segments (simulate.cu); force
    # 256-sample segments so echoes straddle segment edges
    monkeypatch.setenv("KKB_SIM_SEG", "256")
    arr = kb.TransducerArray(24, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    params = kb.AcquisitionParams(C, kb.transmit_angles(3, np.deg2rad(10)), 1024, start_time=1e-6)
    ph = kb.speckle_phantom((-4e-3, 4e-3, 3e-3, 20e-3), 1.0e7, seed=5)
    pulse = kb.make_pulse(5.2e6, 0.3, 20.8e6)  # longer than 32 samples: multi-sample lanes
    assert pulse.waveform.size > 32
    rf = kb.simulate_rf(arr, params, ph, pulse)
    ref = oracle.simulate_rf(arr.positions, params.transmit_angles, C, 1024, 1e-6,
                             arr.sampling_frequency, ph.x, ph.z, ph.reflectivity, pulse.waveform)
    assert np.array_equal(rf.data, ref)
