"""Pin the oracle: every restated function reproduces the golden vectors the
reference itself produced (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import C, DEG, golden, rel_l2, sha


def test_simulator_and_analytic_match_reference_bytes(oracle, config1_rf):
    w, rf = config1_rf
    g = golden("config1")
    an = oracle.analytic_signal(rf)
    assert sha(an) == str(g["an_sha"])


def test_pulse_matches_reference(oracle):
    g = golden("config1")
    assert np.array_equal(oracle.make_pulse(5e6, 0.44, 20e6), g["pulse"])
    assert np.array_equal(oracle.make_pulse(5.2e6, 0.67, 20.83e6), golden("das_point")["pulse"])


def test_analytic_signal_goldens(oracle):
    g = golden("spectral")
    for T in (64, 96, 128, 200, 256, 1536):
        assert np.array_equal(oracle.analytic_signal(g[f"in_{T}"]), g[f"out_{T}"]), T


def test_one_sided_weights_even_odd(oracle):
    w = oracle.one_sided_weights(8)
    assert list(w) == [1, 2, 2, 2, 1, 0, 0, 0]
    w = oracle.one_sided_weights(7)
    assert list(w) == [1, 2, 2, 2, 0, 0, 0]


@pytest.mark.parametrize("T,seed", [(256, 0), (512, 4)])
def test_compress_goldens(oracle, T, seed):
    g = golden("compress")
    rng = np.random.default_rng(seed)
    rf = rng.standard_normal((2, 64, T)).astype(np.float32)
    an = oracle.analytic_signal(rf)
    assert sha(an) == str(g[f"an_sha_{T}"])
    pos = oracle.element_positions(64, 0.23e-3)
    for label in ("vern", "expl"):
        rx = g[f"rx_{label}_{T}"]
        assert np.array_equal(oracle.compress(an, 20.83e6, pos, rx, C), g[f"compress_{label}_{T}"])
        assert np.array_equal(oracle.shear_and_sum(an, 20.83e6, pos, rx, C), g[f"shear_{label}_{T}"])


def test_config1_stage1_and_luts(oracle, config1_rf):
    w, rf = config1_rf
    g = golden("config1")
    fs, pos = w.array.sampling_frequency, w.array.positions
    rfc = oracle.decompose_f64(rf, fs, pos, g["rx"], C)
    assert np.array_equal(rfc, g["compressed"])
    assert np.array_equal(oracle.decompose_c64_staged(rf, fs, pos, g["rx"], C), g["staged_c64"])
    luts = oracle.kk_luts(w.grid.x, w.grid.z, g["tx"], g["rx"], C)
    for a, k in zip(luts, ("ltx", "ltz", "lrx", "lrz")):
        assert np.array_equal(a, g[k]), k


def test_config1_kk_images_bit_exact(oracle, config1_rf):
    w, _ = config1_rf
    g = golden("config1")
    luts = [g[k] for k in ("ltx", "ltz", "lrx", "lrz")]
    fs, t0 = 20e6, 6e-6
    img = oracle.kk_kernel(g["compressed"], *luts, np.ones(11), fs, (0.0 - t0) * fs)
    assert np.array_equal(img, g["image"])
    img = oracle.kk_kernel(g["compressed"], *luts, g["weights"], fs, (0.3e-6 - t0) * fs, linear=False)
    assert np.array_equal(img, g["image_nearest"])
    img = oracle.kk_kernel(g["compressed"], *luts, g["weights"], fs, (-0.2e-6 - t0) * fs)
    assert np.array_equal(img, g["image_weighted"])
    # thread count does not change a bit (criterion 10 analogue)
    img1 = oracle.kk_kernel(g["compressed"], *luts, np.ones(11), fs, (0.0 - t0) * fs, threads=1)
    assert np.array_equal(img1, g["image"])
    # pixel-range evaluation equals the matching slice of the full image
    part = oracle.kk_kernel(g["compressed"], *luts, np.ones(11), fs, (0.0 - t0) * fs,
                            p_range=(1000, 3000))
    assert np.array_equal(part, g["image"].ravel()[1000:3000])


def test_kk_taps_reproduce_image_nearest(oracle):
    # the numpy tap restatement rebuilds the nearest-mode image exactly
    g = golden("config1")
    luts = [g[k] for k in ("ltx", "ltz", "lrx", "lrz")]
    fs, t0 = 20e6, 6e-6
    shift = (0.3e-6 - t0) * fs
    j, ok = oracle.kk_taps(*luts, fs, shift, 1024, linear=False)
    data = g["compressed"]
    w = g["weights"]
    X, Z, N, M = j.shape
    acc = np.zeros((X, Z), np.complex128)
    jc = np.clip(j, 0, 1023)
    for n in range(N):
        for m in range(M):
            vals = data[n, m][jc[:, :, n, m]].astype(np.complex128) * w[m]
            acc += np.where(ok[:, :, n, m], vals, 0)
    assert rel_l2(acc, g["image_nearest"]) < 1e-13


def test_das_goldens(oracle, point_dataset):
    arr, params, rf, grid = point_dataset
    g = golden("das_point")
    an = oracle.analytic_signal(rf)
    assert sha(an) == str(g["an_sha"])
    ltx, ltz, hyp, base, frac = oracle.das_luts(grid.x0, grid.dx, grid.nx, grid.z, arr.positions,
                                               arr.aperture, params.transmit_angles, C)
    assert np.array_equal(hyp, g["hyp"]) and np.array_equal(base, g["base"])
    assert np.array_equal(frac, g["frac"])
    fs = arr.sampling_frequency
    args = (an, ltx, ltz, hyp, base, frac, grid.x, grid.z, arr.positions)
    img = oracle.das_kernel(*args, np.inf, np.ones(64), fs, 0.0)
    assert np.array_equal(img, g["image"])
    img = oracle.das_kernel(*args, np.tan(0.3), np.ones(64), fs, 0.0)
    assert np.array_equal(img, g["image_gated"])
    img = oracle.das_kernel(*args, np.inf, np.ones(64), fs, 0.0, linear=False)
    assert np.array_equal(img, g["image_nearest"])
    assert rel_l2(g["image"], g["image_direct"]) <= 1e-4


@pytest.mark.parametrize("name,cfg", [("config2_noise", 2), ("config4_noise", 4)])
def test_noise_config_goldens(oracle, name, cfg):
    from paper_2603_22496_b200 import configs

    w = configs.CONFIGS[cfg]()
    g = golden(name)
    p, arr = w.params, w.array
    rf = oracle.noise_volume(p.num_transmits, arr.num_elements, p.num_samples, seed=cfg)
    assert sha(rf) == str(g["rf_sha"])
    assert np.array_equal(p.transmit_angles, g["tx"])
    assert np.array_equal(w.receive.angles, g["rx"])
    fs = arr.sampling_frequency
    rfc = oracle.decompose_f64(rf, fs, arr.positions, g["rx"], C)
    assert np.array_equal(rfc, g["compressed"])
    luts = oracle.kk_luts(w.grid.x, w.grid.z, g["tx"], g["rx"], C)
    for a, k in zip(luts, ("ltx", "ltz", "lrx", "lrz")):
        assert np.array_equal(a, g[k]), k
    img = oracle.kk_kernel(rfc, *luts, np.ones(w.receive.num_angles), fs, 0.0)
    assert np.array_equal(img, g["image"])
