"""Parity on the BASELINE media and full sizes.

* config 2: speckle (10 per resolution cell) + two 2 mm anechoic cysts + six
  amplitude-20 wires, rendered by the GPU simulator (bit-identical to the
  reference's _render_traces), int16-quantised; the KK path (15 x 5 pairs,
  int16 ingest) and the full-size DAS comparison (75 tx x 128 elements,
  9.8e8 samples) against the oracle;
* config 4: a 16-frame functional-ultrasound ensemble, static background +
  a 2 mm vessel whose scatterers move 50 um per frame, every frame against
  the oracle;
* config 3: all four sampling schemes on a 4-frame batch;
* config 5: the whole 1024 x 2048 image (961 pairs, 2.0e9 pixel-pairs) on
  the config-5 speckle (20 per cell) against the oracle;
* the delay tables of configs 3 and 5 bit-identical to the reference's.

Tolerances: decomposed traces and IQ rel L2 <= 1e-5 (north star), DAS rel L2
<= 1e-5, delay tables bit-exact; the medium sanity checks (cysts dark,
wires bright, frame differences inside the vessel) are physics, not parity.
"""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import configs  # noqa: E402


@pytest.fixture(scope="module")
def config2_rf75():
    """Config-2 medium rendered for all 75 DAS transmits (noise-free)."""
    w = configs.config2()
    arr = w.array
    das_params = w.extra_receive["das75"][0]
    pulse = kb.make_pulse(arr.center_frequency, arr.fractional_bandwidth, arr.sampling_frequency)
    rf = kb.simulate_rf(arr, das_params, configs.config2_medium(0), pulse).data
    return w, das_params, rf


def _oracle_image(oracle, w, params, rx, rf_f32, linear=True):
    arr, g = w.array, w.grid
    fs, c = arr.sampling_frequency, params.sound_speed
    tr = oracle.decompose_f64(rf_f32, fs, arr.positions, rx.angles, c)
    luts = oracle.kk_luts(g.x, g.z, params.transmit_angles, rx.angles, c)
    shift = (0.0 - params.start_time) * fs
    return tr, oracle.kk_kernel(tr, *luts, np.ones(rx.num_angles), fs, shift, linear)


def test_config2_medium_int16_kk_vs_oracle(oracle, config2_rf75):
    import torch

    w, das_params, rf75 = config2_rf75
    rf = np.ascontiguousarray(rf75[2::5])          # the KK transmits tx75[2::5]
    q, scale = configs.quantize_int16(rf)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    assert np.array_equal(p.transmit_angles, das_params.transmit_angles[2::5])
    eng = kb.KKEngine(arr, p, rx, g, frames=1, want_db=False)
    iq = eng.run(torch.from_numpy(q[None]).cuda())
    torch.cuda.synchronize()
    got_tr, got = eng.traces[0].cpu().numpy(), iq[0].cpu().numpy()
    ref_tr, ref = _oracle_image(oracle, w, p, rx, q.astype(np.float32))
    assert rel_l2(got_tr, ref_tr) <= 1e-5
    assert rel_l2(got, ref) <= 1e-5
    # the medium is what it claims: the brightest echo is a wire (the 15 x 5
    # vernier image is too coarse for the 2 mm cysts; the DAS test checks them)
    I = np.abs(ref) ** 2
    ix, iz = np.unravel_index(np.argmax(I), I.shape)
    assert abs(g.z[iz] - configs.WIRES_C2_DEPTH) < 0.5e-3
    eng.close()


def test_config2_das_full_size_vs_oracle(oracle, config2_rf75):
    """The DAS comparison kernel at the configuration it is quoted on: 75
    transmits x 128 elements onto the 256 x 400 grid (9.8e8 samples)."""
    w, das_params, rf75 = config2_rf75
    arr, g = w.array, w.grid
    an = kb.analytic_signal(kb.RFVolume(rf75, arr, das_params))
    luts = kb.build_das_luts(g, arr, das_params)
    got = kb.das(an, luts).pixels
    ref = oracle.das_kernel(an.data, luts.lut_tx_x, luts.lut_tx_z, luts.lut_rx_hypot, luts.rx_base,
                            luts.rx_frac, g.x, g.z, arr.positions, np.inf,
                            np.ones(arr.num_elements), arr.sampling_frequency, 0.0)
    assert rel_l2(got, ref) <= 1e-5
    # the medium is what it claims: both 2 mm cysts anechoic in the
    # full-aperture image (> 10 dB below the speckle around them)
    I = np.abs(got) ** 2
    X, Z = np.meshgrid(g.x, g.z, indexing="ij")
    for cx, cz in configs.CYSTS_C2:
        r2 = (X - cx) ** 2 + (Z - cz) ** 2
        inside, ring = r2 < (1.2e-3) ** 2, (r2 > (3e-3) ** 2) & (r2 < (5e-3) ** 2)
        assert I[inside].mean() < 0.1 * I[ring].mean(), (cx, cz)


def test_config4_vessel_ensemble_vs_oracle(oracle):
    """16 frames of background + moving vessel, one batched launch, every
    frame against the oracle; frame-to-frame changes sit in the vessel."""
    import torch

    F = 16
    w = configs.config4(frames=F)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    pulse = kb.make_pulse(arr.center_frequency, arr.fractional_bandwidth, arr.sampling_frequency)
    bg = kb.render_rf_device(arr, p, configs.config4_background(0), pulse)
    rf = torch.empty((F,) + tuple(bg.shape), dtype=torch.float32, device="cuda")
    for f in range(F):
        rf[f].copy_(bg)
        kb.render_rf_device(arr, p, configs.config4_vessel_frame(f), pulse, out=rf[f])
    eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False)
    iq = eng.run(rf).cpu().numpy()
    rf_h = rf.cpu().numpy()
    for f in range(F):
        _, ref = _oracle_image(oracle, w, p, rx, rf_h[f])
        assert rel_l2(iq[f], ref) <= 1e-5, f
    # frame-to-frame changes: in the vessel band, not in the static tissue
    # above it (echoes arrive after the vessel's, so the plane-wave
    # decomposition's aperture-truncation tails only reach deeper pixels)
    d = np.abs(np.diff(iq, axis=0)) ** 2
    in_vessel = np.abs(g.z - configs.VESSEL_Z) < 1.5e-3
    above = g.z < configs.VESSEL_Z - 3e-3
    assert d[:, :, in_vessel].mean() > 100 * d[:, :, above].mean()
    eng.close()


def test_config3_schemes_batched_vs_oracle(oracle):
    """The four config-3 schemes on a 4-frame batch of distinct frames."""
    import torch

    base = configs.config3()
    arr, g = base.array, base.grid
    for name, (p, rx) in base.extra_receive.items():
        w = configs.Workload(name, arr, p, rx, g)
        F = 4
        rf = np.stack([configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=90 + f)
                       for f in range(F)])
        eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False)
        iq = eng.run(torch.from_numpy(rf).cuda()).cpu().numpy()
        for f in range(F):
            _, ref = _oracle_image(oracle, w, p, rx, rf[f])
            assert rel_l2(iq[f], ref) <= 1e-5, (name, f)
        eng.close()


@pytest.mark.parametrize("cfg", [3, 5])
def test_delay_tables_bit_identical(oracle, cfg):
    w = configs.CONFIGS[cfg]()
    sets = list(w.extra_receive.values()) if cfg == 3 else [(w.params, w.receive)]
    for p, rx in sets:
        luts = kb.build_kk_luts(w.grid, p, rx)
        ref = oracle.kk_luts(w.grid.x, w.grid.z, p.transmit_angles, rx.angles, p.sound_speed)
        for got, want in zip((luts.lut_tx_x, luts.lut_tx_z, luts.lut_rx_x, luts.lut_rx_z), ref):
            assert np.array_equal(got, want)


def test_config5_full_image_on_speckle_vs_oracle(oracle):
    """The whole config-5 frame (1024 x 2048 pixels, 31 x 31 pairs) on its
    speckle medium (20 scatterers per resolution cell), IQ over every pixel."""
    import torch

    w = configs.config5()
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    a = arr.aperture
    dens = 2.0 * configs.speckle_density(arr, 0.5 * (g.z[0] + g.z[-1]))
    ph = kb.speckle_phantom((-a / 2, a / 2, g.z[0], g.z[-1]), dens, 5)
    pulse = kb.make_pulse(arr.center_frequency, arr.fractional_bandwidth, arr.sampling_frequency)
    rf = kb.render_rf_device(arr, p, ph, pulse)
    eng = kb.KKEngine(arr, p, rx, g, frames=1, want_db=False)
    iq = eng.run(rf[None]).cpu().numpy()[0]
    got_tr = eng.traces[0].cpu().numpy()
    ref_tr, ref = _oracle_image(oracle, w, p, rx, rf.cpu().numpy())
    assert rel_l2(got_tr, ref_tr) <= 1e-5
    assert rel_l2(iq, ref) <= 1e-5
    eng.close()
