"""Seeded random geometries through kk / das / compress against the oracle:
pair counts, trace lengths, grid shapes and spacings, shifts, interpolation
modes and weights drawn at random (edge sizes included: 1 transmit, 1 receive
angle, 1-pixel rows), so the tiled kernels, their fallbacks and the window
sizing meet geometries the fixed configs do not."""

import os

import numpy as np
import pytest

from conftest import C, rel_l2

pytestmark = pytest.mark.gpu

import paper_2603_22496_b200 as kb  # noqa: E402

# KKB_FUZZ_SCALE=k multiplies every case count (a long sweep: scripts/README)
_SCALE = max(1, int(os.environ.get("KKB_FUZZ_SCALE", "1")))


def _sym(rng, m, amax):
    half = np.sort(rng.uniform(0.0, amax, m // 2))
    ang = np.concatenate([-half[::-1], [0.0] if m % 2 else [], half])
    return ang


@pytest.mark.parametrize("seed", range(40 * _SCALE))
def test_kk_random_geometry(oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    n_tx = int(rng.integers(1, 10))
    m_rx = int(rng.integers(1, 13))
    T = int(rng.choice([64, 100, 256, 777, 1024, 1536, 2048]))
    nx, nz = int(rng.integers(1, 90)), int(rng.integers(1, 90))
    fs = float(rng.uniform(10e6, 40e6))
    arr = kb.TransducerArray(16, 0.3e-3, fs / 4, fs, 0.6)
    tx = _sym(rng, n_tx, 0.3) if n_tx > 1 else np.array([float(rng.uniform(-0.2, 0.2))])
    params = kb.AcquisitionParams(C, tx, T, start_time=float(rng.uniform(0, 3e-6)))
    rx = kb.explicit_angles(_sym(rng, m_rx, 0.35))
    dx, dz = float(rng.uniform(0.02e-3, 0.6e-3)), float(rng.uniform(0.02e-3, 0.6e-3))
    grid = kb.ImageGrid(float(rng.uniform(-5e-3, 0)), float(rng.uniform(1e-3, 10e-3)), dx, dz, nx, nz)
    data = (rng.standard_normal((n_tx, m_rx, T)) + 1j * rng.standard_normal((n_tx, m_rx, T))).astype(np.complex64)
    rfc = kb.CompressedRF(data, rx, params, arr)
    luts = kb.build_kk_luts(grid, params, rx)
    linear = bool(rng.integers(0, 2))
    pd = float(rng.uniform(-0.5e-6, 0.5e-6))
    w = rng.uniform(0.2, 2.0, m_rx) if rng.integers(0, 2) else None
    cfg = kb.BeamformConfig(interpolation="linear" if linear else "nearest", pulse_delay=pd,
                            channel_weights=w)
    got = kb.kk(rfc, luts, cfg).pixels
    shift = (pd - params.start_time) * fs
    ref = oracle.kk_kernel(data, luts.lut_tx_x, luts.lut_tx_z, luts.lut_rx_x, luts.lut_rx_z,
                           w if w is not None else np.ones(m_rx), fs, shift, linear=linear)
    if np.abs(ref).max() == 0:
        assert np.abs(got).max() == 0
    else:
        assert rel_l2(got, ref) <= 1e-5, (seed, n_tx, m_rx, T, nx, nz)


@pytest.mark.parametrize("seed", range(20 * _SCALE))
def test_das_random_geometry(oracle, seed):
    rng = np.random.default_rng(2000 + seed)
    n_tx = int(rng.integers(1, 8))
    L = int(rng.integers(2, 40))
    T = int(rng.choice([128, 512, 1000, 2048]))
    nx, nz = int(rng.integers(1, 70)), int(rng.integers(1, 70))
    fs = float(rng.uniform(10e6, 40e6))
    arr = kb.TransducerArray(L, float(rng.uniform(0.1e-3, 0.4e-3)), fs / 4, fs, 0.6)
    tx = _sym(rng, n_tx, 0.3) if n_tx > 1 else np.array([0.1])
    params = kb.AcquisitionParams(C, tx, T, start_time=float(rng.uniform(0, 2e-6)))
    grid = kb.ImageGrid(float(rng.uniform(-4e-3, 0)), float(rng.uniform(1e-3, 8e-3)),
                        float(rng.uniform(0.03e-3, 0.4e-3)), float(rng.uniform(0.03e-3, 0.4e-3)), nx, nz)
    data = (rng.standard_normal((n_tx, L, T)) + 1j * rng.standard_normal((n_tx, L, T))).astype(np.complex64)
    an = kb.AnalyticRF(data, arr, params)
    luts = kb.build_das_luts(grid, arr, params)
    gate = float(rng.uniform(0.1, 0.8)) if rng.integers(0, 2) else None
    linear = bool(rng.integers(0, 2))
    w = rng.uniform(0.2, 2.0, L) if rng.integers(0, 2) else None
    cfg = kb.BeamformConfig(interpolation="linear" if linear else "nearest", max_rx_angle=gate,
                            channel_weights=w)
    got = kb.das(an, luts, cfg).pixels
    ref = oracle.das_kernel(data, luts.lut_tx_x, luts.lut_tx_z, luts.lut_rx_hypot, luts.rx_base,
                            luts.rx_frac, grid.x, grid.z, arr.positions,
                            np.tan(gate) if gate is not None else np.inf,
                            w if w is not None else np.ones(L), fs, -params.start_time * fs,
                            linear=linear)
    if np.abs(ref).max() == 0:
        assert np.abs(got).max() == 0
    else:
        assert rel_l2(got, ref) <= 1e-5, (seed, n_tx, L, T, nx, nz)


@pytest.mark.parametrize("seed", range(10 * _SCALE))
def test_decomposition_random_geometry(oracle, seed):
    # analytic_signal + compress (the accuracy path) and the batched engine
    # decomposition on random element counts, lengths and angle sets
    import torch

    rng = np.random.default_rng(3000 + seed)
    n_tx = int(rng.integers(1, 6))
    L = int(rng.integers(2, 70))
    T = int(rng.choice([96, 250, 512, 1021, 1024, 1536, 2048]))
    m_rx = int(rng.integers(1, 12))
    fs = float(rng.uniform(10e6, 40e6))
    arr = kb.TransducerArray(L, float(rng.uniform(0.1e-3, 0.4e-3)), fs / 4, fs, 0.6)
    params = kb.AcquisitionParams(C, np.linspace(-0.1, 0.1, n_tx), T)
    rx = kb.explicit_angles(_sym(rng, m_rx, 0.3))
    rf = rng.standard_normal((n_tx, L, T)).astype(np.float32)
    ref = oracle.decompose_f64(rf, fs, arr.positions, rx.angles, C)
    an = kb.analytic_signal(kb.RFVolume(rf, arr, params))
    guard = kb.guard_band_samples(arr.aperture, float(np.abs(rx.angles).max()), fs, C)
    if guard > T:  # the reference's guard-band check fires even for sample 0
        from paper_2603_22496_b200.errors import GuardBandError

        with pytest.raises(GuardBandError):
            kb.compress(an, rx, last_used_sample=0)
    got = kb.compress(an, rx, last_used_sample=0 if guard <= T else None).data
    assert rel_l2(got, ref) <= 1e-5, (seed, n_tx, L, T, m_rx)
    grid = kb.ImageGrid(-1e-3, 2e-3, 0.1e-3, 0.1e-3, 4, 4)
    eng = kb.KKEngine(arr, params, rx, grid, frames=2, want_db=False)
    eng.decompose(torch.from_numpy(np.stack([rf, rf])).cuda())
    torch.cuda.synchronize()
    tr = eng.traces.cpu().numpy()
    assert rel_l2(tr[0], ref) <= 1e-5 and np.array_equal(tr[0], tr[1]), (seed, n_tx, L, T, m_rx)
    eng.close()


@pytest.mark.parametrize("seed", range(16 * _SCALE))
def test_kk_batched_and_multiset_random(seed, monkeypatch):
    """Kernel-level properties on random geometries: a batch of F frames
    equals F single-frame launches bit for bit through every tiled instance
    (forced with KKB_KK_INST — these grids are too small for the default
    dispatch to pick the 32 x 64 tiles with two frames per CTA — and checked
    with kkb_kk_last_instance whenever the instance's window fits), and one
    multi-set launch over a random partition of the receive angles equals
    one launch per set (per-set tables, intensities accumulated) bit for bit,
    the multi-set launch also forced onto the two-frames-per-CTA instance."""
    import ctypes

    import torch

    from paper_2603_22496_b200 import _device as dev
    from paper_2603_22496_b200 import _lib
    from paper_2603_22496_b200.beamform import build_kk_luts_device

    rng = np.random.default_rng(4000 + seed)
    n_tx = int(rng.integers(1, 12))
    m_rx = int(rng.integers(2, 14))
    T = int(rng.choice([256, 1000, 1024, 1536, 2048]))
    nx, nz = int(rng.integers(60, 300)), int(rng.integers(60, 300))
    frames = int(rng.integers(2, 6))
    fs = float(rng.uniform(10e6, 40e6))
    tx = rng.uniform(-0.3, 0.3, n_tx)
    rx = rng.uniform(-0.35, 0.35, m_rx)
    dx, dz = float(rng.uniform(0.02e-3, 0.15e-3)), float(rng.uniform(0.02e-3, 0.15e-3))
    grid = kb.ImageGrid(float(rng.uniform(-5e-3, 0)), float(rng.uniform(1e-3, 10e-3)), dx, dz, nx, nz)
    linear = int(rng.integers(0, 2))
    shift = float(rng.uniform(-40, 10))
    w = rng.uniform(0.2, 2.0, m_rx)
    data = torch.complex(torch.randn(frames, n_tx, m_rx, T, generator=torch.Generator().manual_seed(seed)),
                         torch.randn(frames, n_tx, m_rx, T)).to(torch.complex64).cuda()
    P = nx * nz
    s = dev.stream_handle()

    def plan(angles, weights):
        luts = build_kk_luts_device(grid, tx, angles, C)
        wd = dev.to_device(np.ascontiguousarray(weights))
        kp = ctypes.c_void_p()
        _lib.call("kkb_kk_plan_create", dev.ptr(luts["lut_tx_x"]), dev.ptr(luts["lut_tx_z"]),
                  dev.ptr(luts["lut_rx_x"]), dev.ptr(luts["lut_rx_z"]), n_tx, len(angles), T, nx,
                  nz, dev.ptr(wd), fs, shift, linear, s, ctypes.byref(kp))
        return kp, (luts, wd)

    kp, keep = plan(rx, w)
    single = torch.empty((frames, nx, nz), dtype=torch.complex64, device="cuda")
    for f in range(frames):
        _lib.call("kkb_kk_plan_run", kp, dev.ptr(data[f]), 1, 0, dev.ptr(single[f]),
                  _lib.KKB_OUT_C64, P, None, None, s)
    ran = set()
    for inst in ("natural", "big_fr", "big", "mid", "direct"):
        if inst != "natural":
            monkeypatch.setenv("KKB_KK_INST", inst)
        batch = torch.empty((frames, nx, nz), dtype=torch.complex64, device="cuda")
        _lib.call("kkb_kk_plan_run", kp, dev.ptr(data), frames, n_tx * m_rx * T, dev.ptr(batch),
                  _lib.KKB_OUT_C64, P, None, None, s)
        torch.cuda.synchronize()
        ran.add(_lib.KKB_KK_INST_NAMES[_lib.last_instance()])
        monkeypatch.delenv("KKB_KK_INST", raising=False)
        assert torch.equal(batch, single), (seed, inst, n_tx, m_rx, T, nx, nz, frames)
    assert "direct" in ran, ran
    assert _lib.take_device_error() == 0
    monkeypatch.setenv("KKB_KK_INST", "big_fr")

    # random partition of the receive angles into 1..4 contiguous sets
    nsets = int(rng.integers(1, min(4, m_rx) + 1))
    cuts = np.sort(rng.choice(np.arange(1, m_rx), nsets - 1, replace=False)) if nsets > 1 else []
    bounds = [0, *[int(c) for c in cuts], m_rx]
    iq_sets = torch.empty((nsets, frames, nx, nz), dtype=torch.complex64, device="cuda")
    inten = torch.empty((frames, nx, nz), dtype=torch.float32, device="cuda")
    fmax = torch.zeros(frames, dtype=torch.int32, device="cuda")
    b = (ctypes.c_int * len(bounds))(*bounds)
    _lib.call("kkb_kk_plan_run_sets", kp, dev.ptr(data), frames, n_tx * m_rx * T, nsets, b,
              dev.ptr(iq_sets), _lib.KKB_OUT_C64, P, frames * P, dev.ptr(inten), dev.ptr(fmax), 0, s)
    monkeypatch.delenv("KKB_KK_INST")
    ref_i = torch.empty_like(inten)
    ref_m = torch.zeros_like(fmax)
    for j in range(nsets):
        a0, a1 = bounds[j], bounds[j + 1]
        kj, kjk = plan(rx[a0:a1], w[a0:a1])
        iq = torch.empty((frames, nx, nz), dtype=torch.complex64, device="cuda")
        _lib.call("kkb_kk_plan_run_strided", kj, dev.ptr(data) + a0 * T * 8, frames,
                  n_tx * m_rx * T, m_rx * T, dev.ptr(iq), _lib.KKB_OUT_C64, P, dev.ptr(ref_i),
                  dev.ptr(ref_m) if j == nsets - 1 else None,
                  _lib.KKB_RUN_ACCUMULATE_INTENSITY if j else 0, s)
        torch.cuda.synchronize()
        _lib.load().kkb_kk_plan_destroy(kj)
        assert torch.equal(iq, iq_sets[j]), (seed, j, bounds)
    assert torch.equal(ref_i, inten) and torch.equal(ref_m, fmax), (seed, bounds)
    _lib.load().kkb_kk_plan_destroy(kp)
    assert _lib.take_device_error() == 0


@pytest.mark.parametrize("seed", range(12 * _SCALE))
def test_simulator_random_geometry(oracle, seed):
    """K8 forward simulator bit-identical to the C restatement of
    _render_traces on random arrays, angles, windows, pulses and point sets
    (echoes clipped at the window start included); a WindowOverflowError must
    name a geometry whose latest echo really runs past the window."""
    from paper_2603_22496_b200.errors import WindowOverflowError

    rng = np.random.default_rng(5000 + seed)
    L = int(rng.integers(2, 40))
    fs = float(rng.uniform(10e6, 40e6))
    fc = fs * float(rng.uniform(0.15, 0.3))
    arr = kb.TransducerArray(L, float(rng.uniform(0.1e-3, 0.4e-3)), fc, fs, float(rng.uniform(0.3, 0.9)))
    n_tx = int(rng.integers(1, 8))
    tx = _sym(rng, n_tx, 0.3) if n_tx > 1 else np.array([float(rng.uniform(-0.2, 0.2))])
    T = int(rng.choice([256, 500, 1024, 2048]))
    t0 = float(rng.uniform(0, 4e-6))
    params = kb.AcquisitionParams(C, tx, T, start_time=t0)
    n_pts = int(rng.integers(1, 200))
    zmax = (t0 + 0.8 * T / fs) * C / 2.2
    ph = kb.Phantom(rng.uniform(-arr.aperture / 2, arr.aperture / 2, n_pts),
                    rng.uniform(0.5e-3, max(1e-3, zmax), n_pts), rng.standard_normal(n_pts))
    pulse = kb.make_pulse(fc, arr.fractional_bandwidth, fs)
    spread = bool(rng.integers(0, 2))
    try:
        rf = kb.simulate_rf(arr, params, ph, pulse, geometric_spreading=spread)
    except WindowOverflowError:
        # the reference's rule (simulate.py:246-264): latest transmit arrival +
        # farther aperture edge, minus t0, in samples, plus the whole pulse >= T
        tau = max((x * np.sin(a) + z * np.cos(a)) / C for x, z in zip(ph.x, ph.z) for a in tx)
        need = max((max((x * np.sin(a) + z * np.cos(a)) / C for a in tx)
                    + max(np.hypot(x - arr.positions[0], z), np.hypot(x - arr.positions[-1], z)) / C
                    - t0) * fs + pulse.waveform.size for x, z in zip(ph.x, ph.z))
        assert tau > 0 and need >= T, (seed, need, T)
        return
    ref = oracle.simulate_rf(arr.positions, params.transmit_angles, C, T, t0, fs, ph.x, ph.z,
                             ph.reflectivity, pulse.waveform, spread=spread)
    assert np.array_equal(rf.data, ref), (seed, L, n_tx, T, n_pts)


@pytest.mark.parametrize("seed", range(30 * _SCALE))
def test_tensor_core_gather_random(seed, monkeypatch):
    """Random geometries and batch sizes through the tensor-core gather
    (forced, KKB_KK_INST=tc) against the FMA gather (KKB_KK_TC=0): partial
    tiles, tail frame blocks, both tap modes, channel weights, complex64 /
    complex128 IQ, fused intensity (optionally accumulated) and frame max.
    Plans too steep for its 4 x 32 tile must fall back to an FMA instance."""
    import ctypes

    import torch

    from paper_2603_22496_b200 import _device as dev
    from paper_2603_22496_b200 import _lib

    rng = np.random.default_rng(7000 + seed)
    n_tx = int(rng.integers(1, 8))
    m_rx = int(rng.integers(1, 12))
    T = int(rng.choice([128, 256, 777, 1024, 1536]))
    nx, nz = int(rng.integers(1, 80)), int(rng.integers(1, 80))
    F = int(rng.integers(1, 140))
    fs = float(rng.uniform(10e6, 40e6))
    tx = _sym(rng, n_tx, 0.3) if n_tx > 1 else np.array([float(rng.uniform(-0.2, 0.2))])
    params = kb.AcquisitionParams(C, tx, T, start_time=float(rng.uniform(0, 3e-6)))
    rx = kb.explicit_angles(_sym(rng, m_rx, 0.35))
    dx, dz = float(rng.uniform(0.02e-3, 0.3e-3)), float(rng.uniform(0.02e-3, 0.3e-3))
    grid = kb.ImageGrid(float(rng.uniform(-5e-3, 0)), float(rng.uniform(1e-3, 10e-3)), dx, dz, nx, nz)
    luts = kb.build_kk_luts(grid, params, rx)
    linear = bool(rng.integers(0, 2))
    w = rng.uniform(0.2, 2.0, m_rx) if rng.integers(0, 2) else None
    c128 = bool(rng.integers(0, 2))
    accum = bool(rng.integers(0, 2))
    d = [dev.to_device(np.ascontiguousarray(a)) for a in (luts.lut_tx_x, luts.lut_tx_z, luts.lut_rx_x, luts.lut_rx_z)]
    wd = dev.to_device(w) if w is not None else None
    kp = ctypes.c_void_p()
    shift = (0.0 - params.start_time) * fs
    _lib.call("kkb_kk_plan_create", *[x.data_ptr() for x in d], n_tx, m_rx, T, nx, nz, dev.ptr(wd), fs, shift,
              int(linear), dev.stream_handle(), ctypes.byref(kp))
    try:
        g = torch.Generator(device="cuda").manual_seed(seed)
        traces = torch.view_as_complex(torch.randn((F, n_tx, m_rx, T, 2), generator=g, device="cuda"))
        P = nx * nz
        base = torch.rand((F, P), generator=g, device="cuda")
        outs = {}
        for mode in ("tc", "fma"):
            if mode == "tc":
                monkeypatch.setenv("KKB_KK_INST", "tc")
            else:
                monkeypatch.setenv("KKB_KK_TC", "0")
            iq = torch.zeros((F, P), dtype=torch.complex128 if c128 else torch.complex64, device="cuda")
            inten = base.clone()
            fmax = torch.zeros(F, dtype=torch.int32, device="cuda")
            _lib.call("kkb_kk_plan_run_ex", kp, dev.ptr(traces), F, n_tx * m_rx * T, dev.ptr(iq),
                      _lib.KKB_OUT_C128 if c128 else _lib.KKB_OUT_C64, P, dev.ptr(inten), dev.ptr(fmax),
                      _lib.KKB_RUN_ACCUMULATE_INTENSITY if accum else 0, dev.stream_handle())
            torch.cuda.synchronize()
            monkeypatch.delenv("KKB_KK_INST", raising=False)
            monkeypatch.delenv("KKB_KK_TC", raising=False)
            outs[mode] = (_lib.last_instance(), iq, inten, fmax.view(torch.float32))
        assert _lib.take_device_error() == 0
        eligible = int(_lib.load().kkb_kk_plan_tc_ksteps(kp)) > 0
        assert (outs["tc"][0] == _lib.KKB_KK_INST_TC) == eligible, (seed, outs["tc"][0], eligible)
        a, b = outs["tc"], outs["fma"]
        for x, y, tol in ((a[1], b[1], 3e-6), (a[2], b[2], 6e-6)):
            for f in range(F):
                ny = float(torch.linalg.vector_norm(y[f]).item())
                e = float(torch.linalg.vector_norm(x[f] - y[f]).item())
                assert e <= tol * ny + 1e-30, (seed, f, e / max(ny, 1e-30))
        assert bool(((a[3] - b[3]).abs() <= 1e-5 * b[3].abs() + 1e-30).all()), seed
    finally:
        _lib.load().kkb_kk_plan_destroy(kp)
