"""GPU parity: libkkb kernels vs the reference's golden vectors and the oracle.

Tolerances (written per test):
  * delay tables and tap indices: bit-exact;
  * decomposed traces / IQ images: relative L2 <= 1e-5 (north star);
  * the reference's own compress tests: max-abs <= 1e-6 x max (test_compress.py);
  * analytic-signal known answers: the reference's atol (test_spectral.py).
"""

import numpy as np
import pytest

from conftest import C, DEG, golden, rel_l2

pytestmark = pytest.mark.gpu

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import _device as dev  # noqa: E402
from paper_2603_22496_b200 import _lib  # noqa: E402
from paper_2603_22496_b200 import configs  # noqa: E402


def _vol(rows, fs=20.83e6):
    data = np.asarray(rows, np.float32)[None, ...]
    L, T = data.shape[1], data.shape[2]
    arr = kb.TransducerArray(max(L, 2), 0.23e-3, 5.2e6, fs, 0.67)
    if L != arr.num_elements:
        data = np.repeat(data, arr.num_elements, axis=1)
    return kb.RFVolume(data, arr, kb.AcquisitionParams(C, [0.0], T))


# ------------------------------------------------------------------ K1/K3 spectral
@pytest.mark.parametrize("T", [64, 96, 128, 200, 256, 1536])
def test_analytic_signal_matches_reference(T):
    g = golden("spectral")
    x = g[f"in_{T}"]
    arr = kb.TransducerArray(4, 0.23e-3, 5.2e6, 20.83e6, 0.67)
    out = kb.analytic_signal(kb.RFVolume(x, arr, kb.AcquisitionParams(C, [0.0], T))).data
    ref = g[f"out_{T}"]
    assert out.dtype == np.complex64
    assert np.abs(out - ref).max() <= 1e-6 * np.abs(ref).max()


def test_analytic_signal_known_answers():
    T, fs = 256, 20.83e6
    f0 = 16 * fs / T
    t = np.arange(T) / fs
    out = kb.analytic_signal(_vol([np.cos(2 * np.pi * f0 * t)])).data[0, 0]
    assert np.allclose(np.abs(out), 1.0, atol=1e-6)
    assert np.allclose(out, np.exp(2j * np.pi * f0 * t), atol=1e-6)
    out = kb.analytic_signal(_vol([np.full(64, 0.37, np.float32)])).data[0, 0]
    assert np.allclose(out, 0.37, atol=1e-7)
    x = np.zeros(128)
    x[40] = 1.0
    out = kb.analytic_signal(_vol([x])).data[0, 0]
    assert out[40].real == pytest.approx(1.0, abs=1e-6)
    assert np.abs(np.fft.fft(out.astype(np.complex128))[65:]).max() <= 1e-6


def test_analytic_signal_odd_and_prime_lengths(oracle):
    # odd T (no Nyquist bin) and a prime length (direct-DFT kernel)
    for T in (7, 255, 1021):
        x = np.random.default_rng(T).standard_normal((1, 4, T)).astype(np.float32)
        arr = kb.TransducerArray(4, 0.23e-3, 5.2e6, 20.83e6, 0.67)
        out = kb.analytic_signal(kb.RFVolume(x, arr, kb.AcquisitionParams(C, [0.0], T))).data
        ref = oracle.analytic_signal(x)
        assert rel_l2(out, ref) <= 1e-5, T


@pytest.mark.parametrize("T", [1024, 1536, 2048, 4096])
def test_compile_time_fft_lengths(oracle, T):
    # the compile-time radix plans (fft_ct.cu) against numpy, odd trace count
    # so the last real pair is half-empty
    x = np.random.default_rng(T).standard_normal((1, 7, T)).astype(np.float32)
    arr = kb.TransducerArray(7, 0.23e-3, 5.2e6, 20.83e6, 0.67)
    out = kb.analytic_signal(kb.RFVolume(x, arr, kb.AcquisitionParams(C, [0.0], T))).data
    ref = oracle.analytic_signal(x)
    assert rel_l2(out, ref) <= 1e-6, T


def test_analytic_real_part_preserves_input():
    x = np.random.default_rng(0).standard_normal((1, 4, 128)).astype(np.float32)
    arr = kb.TransducerArray(4, 0.23e-3, 5.2e6, 20.83e6, 0.67)
    out = kb.analytic_signal(kb.RFVolume(x, arr, kb.AcquisitionParams(C, [0.0], 128))).data
    assert np.abs(out.real - x).max() <= 1e-6 * np.abs(x).max()


# ------------------------------------------------------------------ K1-K3 compress
@pytest.mark.parametrize("T,seed", [(256, 0), (512, 4)])
def test_compress_matches_reference(oracle, small_array, T, seed):
    g = golden("compress")
    params = kb.AcquisitionParams(C, [0.0, 0.1], T)
    rf = np.random.default_rng(seed).standard_normal((2, 64, T)).astype(np.float32)
    an = kb.AnalyticRF(oracle.analytic_signal(rf), small_array, params)
    for label in ("vern", "expl"):
        rx = kb.explicit_angles(g[f"rx_{label}_{T}"])
        out = kb.compress(an, rx).data
        ref = g[f"compress_{label}_{T}"]
        assert np.abs(out - ref).max() <= 1e-6 * np.abs(ref).max(), label
        sh = kb.shear_and_sum(an.data, small_array.sampling_frequency, small_array.positions,
                              rx.angles, C)
        assert sh.dtype == np.complex128
        assert rel_l2(sh, g[f"shear_{label}_{T}"]) <= 1e-6


def test_zero_receive_angle_is_plain_sum(small_array):
    params = kb.AcquisitionParams(C, [0.0, 0.1], 256)
    rf = kb.RFVolume(np.random.default_rng(0).standard_normal((2, 64, 256)).astype(np.float32),
                     small_array, params)
    an = kb.analytic_signal(rf)
    expect = an.data.astype(np.complex128).sum(axis=1)
    out = kb.compress(an, kb.explicit_angles([0.0]))
    assert np.abs(out.data[:, 0, :] - expect).max() <= 1e-6 * np.abs(expect).max()


def test_compress_zeros_and_metadata(small_array):
    params = kb.AcquisitionParams(C, [0.0, 0.1], 128)
    an = kb.analytic_signal(kb.RFVolume(np.zeros((2, 64, 128), np.float32), small_array, params))
    rx = kb.uniform_vernier_angles(7, 5, 12 * DEG, 1)
    out = kb.compress(an, rx)
    assert out.data.shape == (2, 5, 128) and not out.data.any()
    assert out.data.dtype == np.complex64 and out.receive_angles is rx
    assert out.sampling_frequency == small_array.sampling_frequency


def test_compress_linearity(small_array):
    params = kb.AcquisitionParams(C, [0.0, 0.1], 256)
    rng = np.random.default_rng(6)
    shape = (2, 64, 256)
    ints = lambda: (rng.integers(-1000, 1000, shape) + 1j * rng.integers(-1000, 1000, shape)).astype(np.complex64)
    a = kb.AnalyticRF(ints(), small_array, params)
    b = kb.AnalyticRF(ints(), small_array, params)
    mix = kb.AnalyticRF(2.5 * a.data + b.data, small_array, params)
    rx = kb.uniform_vernier_angles(7, 5, 12 * DEG, 1)
    lhs = kb.compress(mix, rx).data
    rhs = 2.5 * kb.compress(a, rx).data + kb.compress(b, rx).data
    assert np.abs(lhs - rhs).max() <= 1e-6 * np.abs(rhs).max()


def test_compress_mirror_symmetry(oracle, small_array):
    params = kb.AcquisitionParams(C, [0.0, 0.1], 512)
    rf = np.random.default_rng(5).standard_normal((2, 64, 512)).astype(np.float32)
    an = kb.AnalyticRF(oracle.analytic_signal(rf), small_array, params)
    rx = kb.uniform_vernier_angles(7, 5, 12 * DEG, 2)
    out = kb.compress(an, rx)
    flipped = kb.AnalyticRF(np.ascontiguousarray(an.data[:, ::-1, :]), small_array, params)
    rx_neg = kb.explicit_angles(-rx.angles, rx.delta_theta_i)
    out_m = kb.compress(flipped, rx_neg)
    order = [int(np.argmin(np.abs(rx_neg.angles + th))) for th in rx.angles]
    scale = np.abs(out.data).max()
    assert np.abs(out.data - out_m.data[:, order, :]).max() <= 1e-6 * scale


def test_compress_matches_time_domain_shear(oracle):
    # test_compress.py:102-133: spectral shear vs lerp slant-stack, 1e-3 rel RMS
    fs = 40e6
    arr = kb.TransducerArray(48, 0.4e-3, 0.5e6, fs, 0.6)
    params = kb.AcquisitionParams(C, kb.transmit_angles(3, 10 * DEG), 2048)
    wave = oracle.make_pulse(0.5e6, 0.6, fs)
    rf = oracle.simulate_rf(arr.positions, params.transmit_angles, C, 2048, 0.0, fs,
                            np.array([0.0, 2e-3]), np.array([14e-3, 20e-3]), np.array([1.0, 0.7]),
                            wave)
    an = kb.analytic_signal(kb.RFVolume(rf, arr, params))
    rx = kb.uniform_vernier_angles(3, 5, 10 * DEG, 1)
    out = kb.compress(an, rx)
    u = arr.positions
    t = np.arange(2048) / fs
    worst = 0.0
    for m, theta in enumerate(rx.angles):
        for n in range(3):
            ref = np.zeros(2048, np.complex128)
            for l in range(48):
                tau = u[l] * np.sin(theta) / C
                tr = an.data[n, l].astype(np.complex128)
                ref += np.interp(t + tau, t, tr.real, left=0, right=0) + 1j * np.interp(
                    t + tau, t, tr.imag, left=0, right=0)
            err = np.sqrt(np.mean(np.abs(out.data[n, m] - ref) ** 2))
            worst = max(worst, err / np.sqrt(np.mean(np.abs(ref) ** 2)))
    assert worst < 1e-3


# ------------------------------------------------------------------ K4 LUTs + taps
def test_kk_luts_bit_exact():
    g = golden("config1")
    w = configs.config1()
    luts = kb.build_kk_luts(w.grid, w.params, w.receive)
    for name, k in (("lut_tx_x", "ltx"), ("lut_tx_z", "ltz"), ("lut_rx_x", "lrx"), ("lut_rx_z", "lrz")):
        assert np.array_equal(getattr(luts, name), g[k]), name
    assert luts.entry_count == kb.cache_model_entries(w.grid, 11, 11, "kk")
    for cfg, name in ((2, "config2_noise"), (4, "config4_noise")):
        w = configs.CONFIGS[cfg]()
        g = golden(name)
        luts = kb.build_kk_luts(w.grid, w.params, w.receive)
        for nm, k in (("lut_tx_x", "ltx"), ("lut_tx_z", "ltz"), ("lut_rx_x", "lrx"), ("lut_rx_z", "lrz")):
            assert np.array_equal(getattr(luts, nm), g[k]), (cfg, nm)


def test_kk_lut_zero_receive_column():
    params = kb.AcquisitionParams(C, kb.transmit_angles(5, 10 * DEG), 128)
    rx = kb.uniform_vernier_angles(5, 5, 10 * DEG, 0)
    grid = kb.ImageGrid(-1.5e-3, 4e-3, 0.09e-3, 0.12e-3, 20, 15)
    luts = kb.build_kk_luts(grid, params, rx)
    assert np.all(luts.lut_rx_x[:, 2] == 0.0)
    assert np.array_equal(luts.lut_rx_z[:, 2], grid.z / C)
    s, co = np.sin(rx.angles), np.cos(rx.angles)
    assert np.array_equal(luts.lut_rx_x, grid.x[:, None] * s[None, :] / C)
    assert np.array_equal(luts.lut_rx_z, grid.z[:, None] * co[None, :] / C)


@pytest.mark.parametrize("linear,pulse_delay", [(True, 0.0), (False, 0.3e-6), (True, -0.2e-6)])
def test_tap_indices_bit_exact(oracle, linear, pulse_delay):
    g = golden("config1")
    luts = [g[k] for k in ("ltx", "ltz", "lrx", "lrz")]
    fs, t0, T = 20e6, 6e-6, 1024
    shift = (pulse_delay - t0) * fs
    i0, ok = oracle.kk_taps(*luts, fs, shift, T, linear=linear)
    d = [dev.to_device(a) for a in luts]
    X, Z, N, M = i0.shape
    idx = dev.empty((X, Z, N, M), np.int32)
    _lib.call("kkb_kk_taps", *[x.data_ptr() for x in d], N, M, T, X, Z, fs, shift, int(linear),
              idx.data_ptr(), dev.stream_handle())
    got = dev.to_host(idx)
    assert np.array_equal(got >= 0, ok)
    assert np.array_equal(got[ok], i0[ok])


def test_tap_indices_bit_exact_config5_sample(oracle):
    # the largest geometry: 961 pairs, 4096 samples; a 64 x 64 pixel block
    w = configs.config5()
    luts = kb.build_kk_luts(w.grid, w.params, w.receive)
    sl = (slice(480, 544), slice(1000, 1064))
    sub = [luts.lut_tx_x[sl[0]], luts.lut_tx_z[sl[1]], luts.lut_rx_x[sl[0]], luts.lut_rx_z[sl[1]]]
    fs = w.array.sampling_frequency
    i0, ok = oracle.kk_taps(*sub, fs, 0.0, 4096)
    d = [dev.to_device(np.ascontiguousarray(a)) for a in sub]
    X, Z, N, M = i0.shape
    idx = dev.empty((X, Z, N, M), np.int32)
    _lib.call("kkb_kk_taps", *[x.data_ptr() for x in d], N, M, 4096, X, Z, fs, 0.0, 1,
              idx.data_ptr(), dev.stream_handle())
    got = dev.to_host(idx)
    assert np.array_equal(got >= 0, ok) and np.array_equal(got[ok], i0[ok])


# ------------------------------------------------------------------ K5 kk
def _c1_rfc(w, g):
    return kb.CompressedRF(g["compressed"], w.receive, w.params, w.array)


def test_kk_matches_reference_images():
    g = golden("config1")
    w = configs.config1()
    rfc = _c1_rfc(w, g)
    luts = kb.build_kk_luts(w.grid, w.params, w.receive)
    img = kb.kk(rfc, luts).pixels
    assert img.dtype == np.complex128
    assert rel_l2(img, g["image"]) <= 1e-5
    near = kb.kk(rfc, luts, kb.BeamformConfig(interpolation="nearest", pulse_delay=0.3e-6,
                                              channel_weights=g["weights"])).pixels
    assert rel_l2(near, g["image_nearest"]) <= 1e-5
    wtd = kb.kk(rfc, luts, kb.BeamformConfig(pulse_delay=-0.2e-6, channel_weights=g["weights"])).pixels
    assert rel_l2(wtd, g["image_weighted"]) <= 1e-5


@pytest.mark.parametrize("name,cfg", [("config2_noise", 2), ("config4_noise", 4)])
def test_kk_noise_configs_match_reference(name, cfg):
    g = golden(name)
    w = configs.CONFIGS[cfg]()
    rfc = kb.CompressedRF(g["compressed"], w.receive, w.params, w.array)
    luts = kb.build_kk_luts(w.grid, w.params, w.receive)
    img = kb.kk(rfc, luts).pixels
    assert rel_l2(img, g["image"]) <= 1e-5


def test_kk_zero_and_deterministic(small_array):
    params = kb.AcquisitionParams(C, [0.0, 0.1], 256)
    grid = kb.ImageGrid(-1e-3, 5e-3, 0.1e-3, 0.1e-3, 12, 10)
    rx = kb.explicit_angles([-0.1, 0.0, 0.1])
    rfc = kb.CompressedRF(np.zeros((2, 3, 256), np.complex64), rx, params, small_array)
    luts = kb.build_kk_luts(grid, params, rx)
    assert np.all(kb.kk(rfc, luts).pixels == 0.0)
    g = golden("config1")
    w = configs.config1()
    l1 = kb.build_kk_luts(w.grid, w.params, w.receive)
    a = kb.kk(_c1_rfc(w, g), l1).pixels
    b = kb.kk(_c1_rfc(w, g), l1).pixels
    assert np.array_equal(a, b)


def test_kk_geometry_mismatch_rejected(small_array):
    params = kb.AcquisitionParams(C, [0.0, 0.1], 128)
    grid = kb.ImageGrid(-1e-3, 5e-3, 0.1e-3, 0.1e-3, 10, 10)
    rx = kb.explicit_angles([-0.1, 0.0, 0.1])
    rfc = kb.CompressedRF(np.zeros((2, 3, 128), np.complex64), rx, params, small_array)
    kluts = kb.build_kk_luts(grid, params, rx)
    dluts = kb.build_das_luts(grid, small_array, params)
    with pytest.raises(kb.GeometryError):
        kb.kk(rfc, dluts)
    other_rx = kb.explicit_angles([-0.2, 0.0, 0.2])
    with pytest.raises(kb.GeometryError):
        kb.kk(kb.CompressedRF(rfc.data, other_rx, params, small_array), kluts)
    with pytest.raises(kb.GeometryError):
        kb.kk(rfc, kluts, kb.BeamformConfig(channel_weights=np.ones(4)))


def test_kk_many_receive_angles_and_odd_grid(oracle, small_array):
    # 64 receive angles force the receive-chunked pipeline; 37 x 45 grid has partial tiles
    rng = np.random.default_rng(9)
    params = kb.AcquisitionParams(C, kb.transmit_angles(5, 12 * DEG), 1024)
    rx = kb.explicit_angles(np.linspace(-0.3, 0.3, 64))
    data = (rng.standard_normal((5, 64, 1024)) + 1j * rng.standard_normal((5, 64, 1024))).astype(np.complex64)
    grid = kb.ImageGrid(-2e-3, 6e-3, 0.11e-3, 0.07e-3, 37, 45)
    rfc = kb.CompressedRF(data, rx, params, small_array)
    luts = kb.build_kk_luts(grid, params, rx)
    img = kb.kk(rfc, luts).pixels
    ref = oracle.kk_kernel(data, luts.lut_tx_x, luts.lut_tx_z, luts.lut_rx_x, luts.lut_rx_z,
                           np.ones(64), small_array.sampling_frequency, 0.0)
    assert rel_l2(img, ref) <= 1e-5


# ------------------------------------------------------------------ K7 das
def test_das_matches_reference(oracle, point_dataset):
    arr, params, rf, grid = point_dataset
    g = golden("das_point")
    an = kb.AnalyticRF(oracle.analytic_signal(rf), arr, params)
    luts = kb.build_das_luts(grid, arr, params)
    assert np.array_equal(luts.lut_rx_hypot, g["hyp"])
    assert rel_l2(kb.das(an, luts).pixels, g["image"]) <= 1e-5
    assert rel_l2(kb.das(an, luts, kb.BeamformConfig(max_rx_angle=0.3)).pixels, g["image_gated"]) <= 1e-5
    assert rel_l2(kb.das(an, luts, kb.BeamformConfig(interpolation="nearest")).pixels,
                  g["image_nearest"]) <= 1e-5
    assert rel_l2(kb.das(an, luts).pixels, g["image_direct"]) <= 1e-4
    doubled = kb.das(an, luts, kb.BeamformConfig(channel_weights=np.full(64, 2.0))).pixels
    assert np.allclose(doubled, 2.0 * kb.das(an, luts).pixels, rtol=1e-6)


# ------------------------------------------------------------------ K6 detection
def _toy(seed, grid=None):
    grid = grid or kb.ImageGrid(-1e-3, 2e-3, 0.1e-3, 0.1e-3, 8, 6)
    rng = np.random.default_rng(seed)
    return kb.ComplexImage(rng.standard_normal((8, 6)) + 1j * rng.standard_normal((8, 6)), grid)


def test_intensity_and_compounding(oracle):
    im, im2 = _toy(0), _toy(1)
    assert np.allclose(kb.intensity(im).pixels, oracle.intensity(im.pixels), rtol=1e-14)
    assert np.allclose(kb.compound_coherent([im, im2]).pixels,
                       oracle.compound_coherent([im.pixels, im2.pixels]), rtol=1e-13)
    assert np.allclose(kb.compound_incoherent([im, im2]).pixels,
                       oracle.compound_incoherent([im.pixels, im2.pixels]), rtol=1e-13)
    neg = kb.ComplexImage(-im.pixels, im.grid)
    assert np.all(kb.compound_coherent([im, neg]).pixels == 0.0)
    other = kb.ComplexImage(np.zeros((8, 6)), kb.ImageGrid(-1e-3, 3e-3, 0.1e-3, 0.1e-3, 8, 6))
    with pytest.raises(kb.GeometryError):
        kb.compound_coherent([im, other])
    with pytest.raises(kb.ConfigError):
        kb.compound_incoherent([])


@pytest.mark.parametrize("direct", ["0", "1"])
def test_das_odd_grid_gated_weighted_vs_oracle(oracle, small_array, monkeypatch, direct):
    # partial tiles, element groups, the per-tile gate skip, and (direct=1) the
    # per-pixel fallback kernel, against the C restatement of _das_kernel
    monkeypatch.setenv("KKB_DAS_DIRECT", direct)
    rng = np.random.default_rng(21)
    params = kb.AcquisitionParams(C, kb.transmit_angles(7, 12 * DEG), 1024, start_time=1e-6)
    data = (rng.standard_normal((7, 64, 1024)) + 1j * rng.standard_normal((7, 64, 1024))).astype(np.complex64)
    grid = kb.ImageGrid(-3e-3, 5e-3, 0.07e-3, 0.09e-3, 45, 37)
    an = kb.AnalyticRF(data, small_array, params)
    luts = kb.build_das_luts(grid, small_array, params)
    w = rng.uniform(0.5, 1.5, 64)
    fs = small_array.sampling_frequency
    for cfg, linear in ((kb.BeamformConfig(max_rx_angle=0.25, channel_weights=w), True),
                        (kb.BeamformConfig(interpolation="nearest", pulse_delay=0.2e-6), False)):
        got = kb.das(an, luts, cfg).pixels
        tan_max = np.tan(cfg.max_rx_angle) if cfg.max_rx_angle is not None else np.inf
        wts = cfg.channel_weights if cfg.channel_weights is not None else np.ones(64)
        shift = (cfg.pulse_delay - params.start_time) * fs
        ref = oracle.das_kernel(data, luts.lut_tx_x, luts.lut_tx_z, luts.lut_rx_hypot, luts.rx_base,
                                luts.rx_frac, grid.x, grid.z, small_array.positions, tan_max, wts,
                                fs, shift, linear=linear)
        assert rel_l2(got, ref) <= 1e-5, (direct, linear)


def test_kk_steep_geometry_falls_back_to_per_pixel_kernel(oracle, small_array):
    # a coarse grid (1 mm pixels): a 32 x 64 tile spans > 1024 samples, so the
    # tiled kernel cannot stage its windows and the per-pixel kernel runs
    rng = np.random.default_rng(17)
    params = kb.AcquisitionParams(C, kb.transmit_angles(5, 12 * DEG), 4096)
    rx = kb.uniform_vernier_angles(5, 5, 12 * DEG, 0)
    data = (rng.standard_normal((5, 5, 4096)) + 1j * rng.standard_normal((5, 5, 4096))).astype(np.complex64)
    grid = kb.ImageGrid(-20e-3, 2e-3, 1e-3, 1.5e-3, 41, 50)
    rfc = kb.CompressedRF(data, rx, params, small_array)
    luts = kb.build_kk_luts(grid, params, rx)
    d = [dev.to_device(a) for a in (luts.lut_tx_x, luts.lut_tx_z, luts.lut_rx_x, luts.lut_rx_z)]
    import ctypes

    h = ctypes.c_void_p()
    _lib.call("kkb_kk_plan_create", *[x.data_ptr() for x in d], 5, 5, 4096, 41, 50, None,
              small_array.sampling_frequency, 0.0, 1, dev.stream_handle(), ctypes.byref(h))
    assert _lib.load().kkb_kk_plan_window(h) > 1024
    _lib.load().kkb_kk_plan_destroy(h)
    ref = oracle.kk_kernel(data, luts.lut_tx_x, luts.lut_tx_z, luts.lut_rx_x, luts.lut_rx_z,
                           np.ones(5), small_array.sampling_frequency, 0.0)
    assert rel_l2(kb.kk(rfc, luts).pixels, ref) <= 1e-5


def test_kk_per_pixel_kernel_matches_reference(monkeypatch):
    monkeypatch.setenv("KKB_KK_DIRECT", "1")
    g = golden("config1")
    w = configs.config1()
    rfc = _c1_rfc(w, g)
    luts = kb.build_kk_luts(w.grid, w.params, w.receive)
    assert rel_l2(kb.kk(rfc, luts).pixels, g["image"]) <= 1e-5
    near = kb.kk(rfc, luts, kb.BeamformConfig(interpolation="nearest", pulse_delay=0.3e-6,
                                              channel_weights=g["weights"])).pixels
    assert rel_l2(near, g["image_nearest"]) <= 1e-5


def test_kk_ten_thousand_pairs(oracle, small_array):
    # 100 x 100 pairs: the per-tile pair tables outgrow shared memory, so the
    # per-pixel kernel takes over (no size limit on the pair set)
    rng = np.random.default_rng(23)
    params = kb.AcquisitionParams(C, np.linspace(-0.2, 0.2, 100), 512)
    rx = kb.explicit_angles(np.linspace(-0.25, 0.25, 100))
    data = (rng.standard_normal((100, 100, 512)) + 1j * rng.standard_normal((100, 100, 512))).astype(np.complex64)
    grid = kb.ImageGrid(-1e-3, 3e-3, 0.1e-3, 0.08e-3, 21, 19)
    rfc = kb.CompressedRF(data, rx, params, small_array)
    luts = kb.build_kk_luts(grid, params, rx)
    ref = oracle.kk_kernel(data, luts.lut_tx_x, luts.lut_tx_z, luts.lut_rx_x, luts.lut_rx_z,
                           np.ones(100), small_array.sampling_frequency, 0.0)
    assert rel_l2(kb.kk(rfc, luts).pixels, ref) <= 1e-5


@pytest.mark.parametrize("T", [8192, 4099, 8193, 12288, 20000, 10007])
def test_analytic_signal_long_and_awkward_lengths(oracle, T):
    # the largest single-CTA length (8192), a prime factor > 31 (4099: direct
    # DFT), four-step lengths above 8192 (8193 = 3 x 2731, 12288, 20000) and a
    # prime above 8192 (10007: direct DFT)
    x = np.random.default_rng(T).standard_normal((1, 3, T)).astype(np.float32)
    arr = kb.TransducerArray(3, 0.23e-3, 5.2e6, 20.83e6, 0.67)
    out = kb.analytic_signal(kb.RFVolume(x, arr, kb.AcquisitionParams(C, [0.0], T))).data
    assert rel_l2(out, oracle.analytic_signal(x)) <= 1e-5, T


def test_long_trace_decomposition_and_compress(oracle, small_array):
    # T = 12288 (four-step FFT) through compress and the batched engine
    import torch

    T = 12288
    params = kb.AcquisitionParams(C, [0.0, 0.1], T)
    rf = np.random.default_rng(41).standard_normal((2, 64, T)).astype(np.float32)
    rf_gpu = rf.copy()
    rx = kb.uniform_vernier_angles(7, 5, 12 * DEG, 1)
    ref = oracle.decompose_f64(rf, small_array.sampling_frequency, small_array.positions,
                               rx.angles, C)
    an = kb.analytic_signal(kb.RFVolume(rf, small_array, params))
    assert rel_l2(kb.compress(an, rx, last_used_sample=0).data, ref) <= 1e-5
    grid = kb.ImageGrid(-1e-3, 2e-3, 0.1e-3, 0.1e-3, 4, 4)
    eng = kb.KKEngine(small_array, params, rx, grid, frames=1, want_db=False)
    eng.decompose(torch.from_numpy(rf_gpu[None]).cuda())
    torch.cuda.synchronize()
    assert rel_l2(eng.traces[0].cpu().numpy(), ref) <= 1e-5
    eng.close()


def test_analytic_signal_rejects_too_long_traces():
    T = (1 << 20) + 2
    arr = kb.TransducerArray(2, 0.23e-3, 5.2e6, 20.83e6, 0.67)
    vol = kb.RFVolume(np.zeros((1, 2, T), np.float32), arr, kb.AcquisitionParams(C, [0.0], T))
    with pytest.raises(kb.KKBeamError):
        kb.analytic_signal(vol)


def test_small_and_big_tile_instances_are_bit_identical(monkeypatch):
    # the 16 x 16 and the 32 x 64 tile instances (forced, and checked with
    # kkb_kk_last_instance: a 4-frame config-4 batch alone dispatches to the
    # 32 x 64 tiles with one frame per CTA); the per-pixel sums run in the
    # same order, so the images agree bit for bit
    import torch

    w = configs.config4(frames=4)
    p, arr = w.params, w.array
    rf = np.stack([configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=s)
                   for s in range(4)])
    eng = kb.KKEngine(arr, p, w.receive, w.grid, frames=4, want_db=False)
    monkeypatch.setenv("KKB_KK_INST", "big")
    big = eng.run(torch.from_numpy(rf).cuda()).clone()
    torch.cuda.synchronize()
    assert _lib.last_instance() == _lib.KKB_KK_INST_BIG
    monkeypatch.setenv("KKB_KK_INST", "small")
    small = eng.run(torch.from_numpy(rf).cuda()).clone()
    torch.cuda.synchronize()
    assert _lib.last_instance() == _lib.KKB_KK_INST_SMALL
    assert torch.equal(big, small)
    eng.close()
