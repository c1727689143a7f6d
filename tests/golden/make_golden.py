"""Generate the golden vectors by running the REFERENCE itself.

Run in the build container (the reference lives at /root/reference, which
the GPU box does not have):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Each case stores the reference's outputs plus SHA-256 digests of its inputs;
inputs are regenerated at test time from seeds (numpy PCG64) or by the
oracle simulator, and the digests prove they are the same bytes.  Outputs
are stored at full precision (complex128 images, complex64 traces), so the
oracle is pinned bit-for-bit where the reference is deterministic.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
DEG = np.pi / 180.0
C = 1540.0


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def save(name, **arrays):
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1e3:.1f} kB")


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF_SRC)
    import kkbeam as kb  # noqa: E402  (the reference, read-only)

    # ---------------------------------------------------------- sampling
    d75 = 32 * DEG / 74
    sets = {
        "tx_11_10": kb.transmit_angles(11, 10 * DEG),
        "tx_75_16": kb.transmit_angles(75, 16 * DEG),
        "tx_31_15": kb.transmit_angles(31, 15 * DEG),
        "vern_11_11_10_0": kb.uniform_vernier_angles(11, 11, 10 * DEG, 0).angles,
        "vern_15_5_35d_7": kb.uniform_vernier_angles(15, 5, 35 * d75, 7).angles,
        "vern_9_9_36d_0": kb.uniform_vernier_angles(9, 9, 36 * d75, 0).angles,
        "vern_7_4_12_1": kb.uniform_vernier_angles(7, 4, 12 * DEG, 1).angles,
        "vern_15_19_24_6": kb.uniform_vernier_angles(15, 19, 24 * DEG, 6).angles,
        "conf_15_21_12": kb.confocal_angles(15, 21, 12 * DEG).angles,
        "conf_31_31_15": kb.confocal_angles(31, 31, 15 * DEG).angles,
        "conf_15_5_35d": kb.confocal_angles(15, 5, 35 * d75).angles,
        "conf_25_3_36d": kb.confocal_angles(25, 3, 36 * d75).angles,
        "vern_25_2_36d_0": kb.uniform_vernier_angles(25, 2, 36 * d75, 0).angles,
    }
    save("sampling", **sets)

    # ---------------------------------------------------------- spectral
    spec = {}
    for T in (64, 96, 128, 200, 256, 1536):
        rng = np.random.default_rng(T)
        x = rng.standard_normal((1, 4, T)).astype(np.float32)
        arr = kb.TransducerArray(4, 0.23e-3, 5.2e6, 20.83e6, 0.67)
        params = kb.AcquisitionParams(C, [0.0], T)
        out = kb.analytic_signal(kb.RFVolume(x, arr, params)).data
        spec[f"in_{T}"] = x
        spec[f"out_{T}"] = out
    save("spectral", **spec)

    # ---------------------------------------------------------- compress (small_array)
    small = kb.TransducerArray(64, 0.23e-3, 5.2e6, 20.83e6, 0.67)
    comp = {}
    for T, seed in ((256, 0), (512, 4)):
        params = kb.AcquisitionParams(C, [0.0, 0.1], T)
        rng = np.random.default_rng(seed)
        rf = kb.RFVolume(rng.standard_normal((2, 64, T)).astype(np.float32), small, params)
        an = kb.analytic_signal(rf)
        comp[f"an_sha_{T}"] = np.array(sha(an.data))
        for label, rx in (("vern", kb.uniform_vernier_angles(7, 5, 12 * DEG, 1)),
                          ("expl", kb.explicit_angles([-7 * DEG, 0.0, 7 * DEG]))):
            comp[f"rx_{label}_{T}"] = rx.angles
            comp[f"compress_{label}_{T}"] = kb.compress(an, rx).data
            comp[f"shear_{label}_{T}"] = kb.shear_and_sum(
                an.data, small.sampling_frequency, small.positions, rx.angles, C)
    save("compress", **comp)

    # ---------------------------------------------------------- config 1 (point targets)
    arr = kb.TransducerArray(64, 0.3e-3, 5e6, 20e6, 0.44)
    tmax = 10 * DEG
    params = kb.AcquisitionParams(C, kb.transmit_angles(11, tmax), 1024, start_time=6e-6)
    rx = kb.uniform_vernier_angles(11, 11, tmax, 0)
    grid = kb.ImageGrid(-9.6e-3, 5e-3, 19.2e-3 / 127, 40e-3 / 127, 128, 128)
    rng = np.random.default_rng(0)
    px = rng.uniform(-8e-3, 8e-3, 5)
    pz = rng.uniform(10e-3, 40e-3, 5)
    phantom = kb.Phantom(px, pz, np.ones(5))
    pulse = kb.make_pulse(5e6, 0.44, 20e6)
    rf = kb.simulate_rf(arr, params, phantom, pulse, noise_rms=1e-3, seed=0)
    an = kb.analytic_signal(rf)
    rfc = kb.compress(an, rx)
    luts = kb.build_kk_luts(grid, params, rx)
    img = kb.kk(rfc, luts)
    w = np.random.default_rng(7).uniform(0.5, 1.5, rx.num_angles)
    bnear = kb.BeamformConfig(interpolation="nearest", pulse_delay=0.3e-6, channel_weights=w)
    img_near = kb.kk(rfc, luts, bnear)
    bw = kb.BeamformConfig(pulse_delay=-0.2e-6, channel_weights=w)
    img_w = kb.kk(rfc, luts, bw)
    # fused complex64 stage-1 form of the reference benchmark
    from kkbeam.bench import _kk_stage_fns
    fns = dict(_kk_stage_fns(rf, rx, luts, kb.BeamformConfig()))
    st = {}
    for name in ("reorg_fft", "hilbert_compress", "ifft"):
        fns[name](st)
    save("config1",
         pulse=pulse.waveform, phantom_x=px, phantom_z=pz,
         rf_sha=np.array(sha(rf.data)), an_sha=np.array(sha(an.data)),
         rx=rx.angles, tx=params.transmit_angles,
         compressed=rfc.data, staged_c64=st["iq"],
         ltx=luts.lut_tx_x, ltz=luts.lut_tx_z, lrx=luts.lut_rx_x, lrz=luts.lut_rx_z,
         image=img.pixels, weights=w, image_nearest=img_near.pixels, image_weighted=img_w.pixels,
         )

    # ---------------------------------------------------------- das point dataset
    pulse52 = kb.make_pulse(5.2e6, 0.67, 20.83e6)
    params7 = kb.AcquisitionParams(C, kb.transmit_angles(7, np.deg2rad(12)), 1024)
    ph3 = kb.Phantom(np.array([0.0, 1.1e-3, -0.9e-3]), np.array([9e-3, 11e-3, 12.5e-3]),
                     np.array([1.0, 0.7, 0.9]))
    rf7 = kb.simulate_rf(small, params7, ph3, pulse52)
    an7 = kb.analytic_signal(rf7)
    dx = 0.23e-3 / 4
    grid7 = kb.ImageGrid(-32 * dx + dx / 2, 7e-3, dx, 0.1e-3, 64, 64)
    dl = kb.build_das_luts(grid7, small, params7)
    save("das_point",
         pulse=pulse52.waveform, rf_sha=np.array(sha(rf7.data)), an_sha=np.array(sha(an7.data)),
         hyp=dl.lut_rx_hypot, base=dl.rx_base, frac=dl.rx_frac,
         image=kb.das(an7, dl).pixels,
         image_gated=kb.das(an7, dl, kb.BeamformConfig(max_rx_angle=0.3)).pixels,
         image_nearest=kb.das(an7, dl, kb.BeamformConfig(interpolation="nearest")).pixels,
         image_direct=kb.direct_das(an7, grid7).pixels)

    # ---------------------------------------------------------- config 2 / config 4 shapes (noise)
    def noise_case(name, arr, params, rx, grid, seed):
        rf = kb.noise_volume(arr, params, seed=seed)
        an = kb.analytic_signal(rf)
        rfc = kb.compress(an, rx)
        luts = kb.build_kk_luts(grid, params, rx)
        img = kb.kk(rfc, luts)
        save(name, rf_sha=np.array(sha(rf.data)), rx=rx.angles, tx=params.transmit_angles,
             compressed=rfc.data, image=img.pixels,
             ltx=luts.lut_tx_x, ltz=luts.lut_tx_z, lrx=luts.lut_rx_x, lrz=luts.lut_rx_z)

    arr2 = kb.TransducerArray(128, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    tx75 = kb.transmit_angles(75, 16 * DEG)
    dd = tx75[1] - tx75[0]
    p2 = kb.AcquisitionParams(C, tx75[2::5], 2048)
    rx2 = kb.explicit_angles(dd * np.array([-2.0, -1.0, 0.0, 1.0, 2.0]), dd)
    a = arr2.aperture
    g2 = kb.ImageGrid(-a / 2, 5e-3, a / 255, (C / 5.2e6) / 4, 256, 400)
    noise_case("config2_noise", arr2, p2, rx2, g2, seed=2)

    p4 = kb.AcquisitionParams(C, kb.transmit_angles(11, 10 * DEG), 1536)
    rx4 = kb.uniform_vernier_angles(11, 11, 10 * DEG, 0)
    g4 = kb.ImageGrid(-a / 2, 5e-3, a / 255, (C / 5.2e6) / 4, 256, 256)
    noise_case("config4_noise", arr2, p4, rx4, g4, seed=4)


if __name__ == "__main__":
    main()
