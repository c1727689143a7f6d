"""GPU parity of the device-resident batched pipeline (KKEngine) on the five
workloads.  Tolerances: traces and IQ rel L2 <= 1e-5 vs the oracle /
reference goldens; batch/rerun results bit-identical."""

import numpy as np
import pytest

from conftest import C, golden, rel_l2, sha

pytestmark = pytest.mark.gpu

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import configs  # noqa: E402


def _torch():
    import torch

    return torch


def _engine(w, frames, **kw):
    return kb.KKEngine(w.array, w.params, w.receive, w.grid, frames=frames, **kw)


def test_engine_config1_point_targets(oracle, config1_rf):
    torch = _torch()
    w, rf = config1_rf
    g = golden("config1")
    eng = _engine(w, 1)
    iq = eng.run(torch.from_numpy(rf[None]).cuda())
    torch.cuda.synchronize()
    assert rel_l2(eng.traces[0].cpu().numpy(), g["compressed"]) <= 1e-5
    assert rel_l2(iq[0].cpu().numpy(), g["image"]) <= 1e-5
    # fused detection + dB map
    inten = eng.inten[0].cpu().numpy().astype(np.float64)
    ref_i = oracle.intensity(g["image"])
    assert rel_l2(inten, ref_i) <= 1e-5
    db = eng.db[0].cpu().numpy()
    ref_db = oracle.log_compress_db(ref_i, floor_db=-60.0)
    assert np.abs(db - ref_db).max() <= 1e-3
    eng.close()


@pytest.mark.parametrize("name,cfg", [("config2_noise", 2), ("config4_noise", 4)])
def test_engine_noise_configs_match_reference(oracle, name, cfg):
    torch = _torch()
    w = configs.CONFIGS[cfg]()
    g = golden(name)
    p, arr = w.params, w.array
    rf = configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=cfg)
    assert sha(rf) == str(g["rf_sha"])
    eng = _engine(w, 1)
    iq = eng.run(torch.from_numpy(rf[None]).cuda())
    torch.cuda.synchronize()
    assert rel_l2(eng.traces[0].cpu().numpy(), g["compressed"]) <= 1e-5
    assert rel_l2(iq[0].cpu().numpy(), g["image"]) <= 1e-5
    eng.close()


def test_engine_batch_equals_single_frames_and_is_deterministic():
    torch = _torch()
    w = configs.config4(frames=6)
    p, arr = w.params, w.array
    rf = np.stack([configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=s)
                   for s in range(6)])
    rf_d = torch.from_numpy(rf).cuda()
    eng = _engine(w, 6, chunk_frames=4)
    a = eng.run(rf_d).clone()
    b = eng.run(rf_d).clone()
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    one = _engine(w, 1)
    for f in (0, 5):
        s = one.run(rf_d[f:f + 1].contiguous()).clone()
        torch.cuda.synchronize()
        assert torch.equal(s[0], a[f])
    eng.close()
    one.close()


def test_engine_run_host_equals_device_path():
    torch = _torch()
    w = configs.config4(frames=5)
    p, arr = w.params, w.array
    rf = np.stack([configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=10 + s)
                   for s in range(5)])
    eng = _engine(w, 5)
    ref = eng.run(torch.from_numpy(rf).cuda()).clone()
    torch.cuda.synchronize()
    host_in = torch.from_numpy(rf).pin_memory()
    host_out = torch.empty((5, w.grid.nx, w.grid.nz), dtype=torch.complex64).pin_memory()
    eng.run_host(host_in, host_out, chunk_frames=2)
    assert torch.equal(host_out, ref.cpu())
    eng.close()


def test_engine_rejects_malformed_inputs():
    """Wrong dtype / shape / device / layout raise ConfigError before any launch."""
    torch = _torch()
    from paper_2603_22496_b200.errors import ConfigError

    w = configs.config1()
    p, arr = w.params, w.array
    eng = _engine(w, 2)
    shape = (2, p.num_transmits, arr.num_elements, p.num_samples)
    good = torch.zeros(shape, dtype=torch.float32, device="cuda")
    for bad in (good.double(), good[:, :, :-1], good.cpu(), good.transpose(2, 3).contiguous().transpose(2, 3),
                good[:1]):
        with pytest.raises(ConfigError):
            eng.run(bad)
    with pytest.raises(ConfigError):
        eng.decompose(good, n_frames=3)
    with pytest.raises(ConfigError):
        eng.run_host(good, torch.empty((2, w.grid.nx, w.grid.nz), dtype=torch.complex64))
    with pytest.raises(ConfigError):
        eng.run_host(good.cpu(), torch.empty((2, w.grid.nx, w.grid.nz), dtype=torch.complex128))
    eng.run(good)
    torch.cuda.synchronize()
    eng.close()


@pytest.mark.parametrize("scheme", ["dense_vernier", "shifted_vernier", "confocal", "hybrid"])
def test_engine_config3_schemes(oracle, scheme):
    torch = _torch()
    w3 = configs.config3()
    params, rx = w3.extra_receive[scheme]
    arr, grid = w3.array, w3.grid
    rf = configs.noise_rf(params.num_transmits, arr.num_elements, params.num_samples, seed=3)
    eng = kb.KKEngine(arr, params, rx, grid, frames=1)
    iq = eng.run(torch.from_numpy(rf[None]).cuda())
    torch.cuda.synchronize()
    fs = arr.sampling_frequency
    ref_tr = oracle.decompose_f64(rf, fs, arr.positions, rx.angles, C)
    assert rel_l2(eng.traces[0].cpu().numpy(), ref_tr) <= 1e-5
    luts = oracle.kk_luts(grid.x, grid.z, params.transmit_angles, rx.angles, C)
    ref = oracle.kk_kernel(ref_tr, *luts, np.ones(rx.num_angles), fs, 0.0)
    assert rel_l2(iq[0].cpu().numpy(), ref) <= 1e-5
    eng.close()


def test_engine_config5_full_size(oracle):
    """Config 5 at full size (961 pairs, 2048 x 1024 px, T = 4096): traces vs the
    float64 oracle over the whole frame, IQ vs the oracle on a row block, and
    linearity over the whole image (size-independent property)."""
    torch = _torch()
    w = configs.config5()
    p, arr, grid = w.params, w.array, w.grid
    rf = configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=5)
    eng = _engine(w, 1)
    iq = eng.run(torch.from_numpy(rf[None]).cuda()).clone()
    torch.cuda.synchronize()
    fs = arr.sampling_frequency
    ref_tr = oracle.decompose_f64(rf, fs, arr.positions, w.receive.angles, C)
    got_tr = eng.traces[0].cpu().numpy()
    assert rel_l2(got_tr, ref_tr) <= 1e-5
    luts = oracle.kk_luts(grid.x, grid.z, p.transmit_angles, w.receive.angles, C)
    rows = (500 * grid.nz, 502 * grid.nz)  # two lateral columns x all depths
    ref = oracle.kk_kernel(ref_tr, *luts, np.ones(31), fs, 0.0, p_range=rows)
    got = iq[0].cpu().numpy().ravel()[rows[0]:rows[1]]
    assert rel_l2(got, ref) <= 1e-5
    # linearity: IQ(2 rf + rf') = 2 IQ(rf) + IQ(rf')
    rf2 = configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=55)
    b = eng.run(torch.from_numpy(rf2[None]).cuda()).clone()
    mix = eng.run(torch.from_numpy((2 * rf + rf2)[None]).cuda()).clone()
    torch.cuda.synchronize()
    assert rel_l2(mix.cpu().numpy(), (2 * iq + b).cpu().numpy()) <= 1e-5
    eng.close()


def test_engine_weights_and_nearest(oracle, config1_rf):
    torch = _torch()
    w, rf = config1_rf
    g = golden("config1")
    eng = kb.KKEngine(w.array, w.params, w.receive, w.grid, frames=1, interpolation="nearest",
                      pulse_delay=0.3e-6, channel_weights=g["weights"])
    iq = eng.run(torch.from_numpy(rf[None]).cuda())
    torch.cuda.synchronize()
    assert rel_l2(iq[0].cpu().numpy(), g["image_nearest"]) <= 1e-5
    eng.close()


def test_engine_int16_ingest_other_lengths():
    # lengths without a compile-time FFT plan widen int16 to float32 first
    torch = _torch()
    arr = kb.TransducerArray(32, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    rx = kb.uniform_vernier_angles(3, 3, 0.1, 0)
    grid = kb.ImageGrid(-1e-3, 3e-3, 0.1e-3, 0.1e-3, 16, 16)
    for T in (777, 1021, 3000):
        p = kb.AcquisitionParams(C, kb.transmit_angles(3, 0.1), T)
        q = np.random.default_rng(T).integers(-30000, 30000, (2, 3, 32, T)).astype(np.int16)
        eng = kb.KKEngine(arr, p, rx, grid, frames=2, want_db=False)
        a = eng.run(torch.from_numpy(q.astype(np.float32)).cuda()).clone()
        b = eng.run(torch.from_numpy(q).cuda()).clone()
        torch.cuda.synchronize()
        assert torch.equal(a, b), T
        eng.close()


@pytest.mark.parametrize("cfg", [1, 2, 4, 5])
def test_engine_int16_ingest_is_exact(cfg):
    """int16-quantised RF (BASELINE config 2) through the int16 ingest path is
    bit-identical to the float32 path on q.astype(float32)."""
    torch = _torch()
    w = configs.CONFIGS[cfg]() if cfg != 4 else configs.config4(frames=3)
    p, arr = w.params, w.array
    frames = 1 if cfg == 5 else 3
    rf = np.stack([configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=s)
                   for s in range(frames)])
    scale = np.abs(rf).max() / 32767.0
    q = np.clip(np.round(rf / scale), -32767, 32767).astype(np.int16)
    eng = _engine(w, frames)
    a = eng.run(torch.from_numpy(q.astype(np.float32)).cuda()).clone()
    ta = eng.traces.clone()
    b = eng.run(torch.from_numpy(q).cuda()).clone()
    tb = eng.traces.clone()
    torch.cuda.synchronize()
    assert torch.equal(ta, tb)
    assert torch.equal(a, b)
    host_in = torch.from_numpy(q).pin_memory()
    host_out = torch.empty(a.shape, dtype=torch.complex64).pin_memory()
    eng.run_host(host_in, host_out, chunk_frames=max(1, frames - 1))
    assert torch.equal(host_out, a.cpu())
    eng.close()


def _oracle_image(oracle, w, rf, rx):
    arr, p, g = w.array, w.params, w.grid
    fs = arr.sampling_frequency
    tr = oracle.decompose_f64(rf, fs, arr.positions, rx.angles, p.sound_speed)
    luts = oracle.kk_luts(g.x, g.z, p.transmit_angles, rx.angles, p.sound_speed)
    shift = oracle.kk_resolved_shift(0.0, p.start_time, fs)
    return oracle.kk_kernel(tr, *luts, np.ones(rx.num_angles), fs, shift)


@pytest.mark.parametrize("mode", ["incoherent", "coherent"])
def test_multiset_compounding_matches_oracle(oracle, config1_rf, mode):
    # a hybrid acquisition: two receive sets over one RF batch (cli.py:250-266)
    torch = _torch()
    w, rf = config1_rf
    tmax = 10 * np.pi / 180
    sets = [kb.uniform_vernier_angles(11, 5, tmax, 0), kb.confocal_angles(11, 3, tmax)]
    eng = kb.MultiSetEngine(w.array, w.params, sets, w.grid, 2, mode=mode)
    inten = eng.run(torch.from_numpy(np.stack([rf, rf])).cuda())
    torch.cuda.synchronize()
    imgs = [_oracle_image(oracle, w, rf, s) for s in sets]
    ref = oracle.compound_incoherent(imgs) if mode == "incoherent" else oracle.compound_coherent(imgs)
    got = inten.cpu().numpy().astype(np.float64)
    assert rel_l2(got[0], ref) <= 1e-5 and rel_l2(got[1], ref) <= 1e-5
    assert np.isclose(float(got[0].max()), float(eng.fmax[0].cpu().numpy().view(np.float32)), rtol=0)
    db = eng.db[0].cpu().numpy()
    assert np.abs(db - oracle.log_compress_db(ref, floor_db=-60.0)).max() <= 1e-3
    if mode == "incoherent":  # per-set images from rows of the shared decomposition
        for j, img in enumerate(imgs):
            assert rel_l2(eng.iq[j][1].cpu().numpy(), img) <= 1e-5, j
    eng.close()


@pytest.mark.parametrize("cfg,interp,direct,mch", [(1, "linear", "0", ""), (1, "nearest", "0", ""),
                                                    (1, "linear", "1", ""), (1, "linear", "0", "2"),
                                                    (3, "linear", "0", ""), (3, "nearest", "0", "1"),
                                                    (5, "linear", "0", "")])
def test_multiset_one_launch_equals_per_set_launches(monkeypatch, cfg, interp, direct, mch):
    """kkb_kk_plan_run_sets (one launch, tables staged once) against one
    strided launch per set over the same shared traces, accumulating the
    intensity: IQ of every set, the compounded intensity and its max are
    bit-identical (tiled kernels; and the per-pixel kernels, KKB_KK_DIRECT=1).
    Config 1 x 3 frames runs the small-tile instance, config 3's hybrid sets x
    4 frames the big-tile one (whose per-set launches run two frames per CTA)."""
    import ctypes

    torch = _torch()
    from paper_2603_22496_b200 import _device as dev
    from paper_2603_22496_b200 import _lib
    from paper_2603_22496_b200.beamform import build_kk_luts_device

    monkeypatch.setenv("KKB_KK_DIRECT", direct)
    if mch:  # sets spanning several receive chunks per stage
        monkeypatch.setenv("KKB_KK_MCH", mch)
    if cfg == 1:
        w = configs.config1()
        p, arr, g = w.params, w.array, w.grid
        tmax = 10 * np.pi / 180
        sets = [kb.uniform_vernier_angles(11, 5, tmax, 0), kb.confocal_angles(11, 3, tmax),
                kb.uniform_vernier_angles(11, 2, tmax, 1)]
        frames = 3
    elif cfg == 3:
        w = configs.config3()
        p, arr, g = w.extra_receive["hybrid"][0], w.array, w.grid
        d = p.transmit_angles[1] - p.transmit_angles[0]
        sets = [kb.confocal_angles(25, 3, 12 * d), kb.uniform_vernier_angles(25, 2, 12 * d, 0)]
        frames = 4
    else:  # config 5 geometry: wide windows, so each set spans several receive chunks
        w = configs.config5()
        p, arr, g = w.params, w.array, w.grid
        tmax = 15 * np.pi / 180
        sets = [kb.confocal_angles(31, 9, tmax), kb.uniform_vernier_angles(31, 7, tmax, 0)]
        frames = 1
    rf = torch.from_numpy(np.stack([configs.noise_rf(p.num_transmits, arr.num_elements,
                                                     p.num_samples, seed=50 + f)
                                    for f in range(frames)])).cuda()
    weights = np.linspace(0.5, 1.5, sum(s.num_angles for s in sets))
    eng = kb.MultiSetEngine(arr, p, sets, g, frames, mode="incoherent", interpolation=interp,
                            channel_weights=weights)
    eng.run(rf)
    torch.cuda.synchronize()
    e = eng.engine
    P = g.nx * g.nz
    inten = torch.empty_like(eng.inten)
    fmax = torch.zeros_like(eng.fmax)
    off = 0
    for j, rs in enumerate(sets):
        luts = build_kk_luts_device(g, p.transmit_angles, rs.angles, p.sound_speed)
        wj = dev.to_device(weights[off:off + rs.num_angles].copy())
        kp = ctypes.c_void_p()
        _lib.call("kkb_kk_plan_create", dev.ptr(luts["lut_tx_x"]), dev.ptr(luts["lut_tx_z"]),
                  dev.ptr(luts["lut_rx_x"]), dev.ptr(luts["lut_rx_z"]), e.N, rs.num_angles, e.T,
                  g.nx, g.nz, dev.ptr(wj), float(e.fs), float(e.shift), int(interp == "linear"),
                  dev.stream_handle(), ctypes.byref(kp))
        iq = torch.empty((frames, g.nx, g.nz), dtype=torch.complex64, device="cuda")
        _lib.call("kkb_kk_plan_run_strided", kp, dev.ptr(e.traces) + off * e.T * 8, frames,
                  e.N * e.M * e.T, e.M * e.T, dev.ptr(iq), _lib.KKB_OUT_C64, P, dev.ptr(inten),
                  dev.ptr(fmax) if j == len(sets) - 1 else None,
                  _lib.KKB_RUN_ACCUMULATE_INTENSITY if j else 0, dev.stream_handle())
        torch.cuda.synchronize()
        _lib.load().kkb_kk_plan_destroy(kp)
        assert torch.equal(iq, eng.iq[j]), j
        off += rs.num_angles
    assert torch.equal(inten, eng.inten)
    assert torch.equal(fmax, eng.fmax)
    eng.close()


def test_run_sets_rejects_bad_bounds():
    import ctypes

    from paper_2603_22496_b200 import _lib
    from paper_2603_22496_b200.errors import ConfigError

    w = configs.config1()
    eng = _engine(w, 1)
    M = eng.M
    for b in ([0, M - 1], [1, M], [0, 5, 5, M], [0] + list(range(1, 10)) + [M]):
        arr = (ctypes.c_int * len(b))(*b)
        with pytest.raises(ConfigError):
            _lib.call("kkb_kk_plan_run_sets", eng._kk, None, 1, 0, len(b) - 1, arr, None, 0, 0, 0,
                      None, None, 0, None)
    eng.close()


@pytest.mark.parametrize("cfg", [1, 4])
def test_engine_graph_replay_equals_eager(cfg):
    """KKEngine.capture: one CUDA graph of the whole path; replays on new RF
    written into the static buffer give the eager result bit for bit."""
    torch = _torch()
    w = configs.CONFIGS[cfg]()
    p, arr = w.params, w.array
    frames = 2
    eng = _engine(w, frames)
    rf = torch.empty((frames, p.num_transmits, arr.num_elements, p.num_samples),
                     dtype=torch.float32, device="cuda")
    rf.copy_(torch.from_numpy(np.stack([configs.noise_rf(p.num_transmits, arr.num_elements,
                                                         p.num_samples, seed=70 + f)
                                        for f in range(frames)])))
    g = eng.capture(rf)
    for seed in (80, 90):
        new = torch.from_numpy(np.stack([configs.noise_rf(p.num_transmits, arr.num_elements,
                                                          p.num_samples, seed=seed + f)
                                         for f in range(frames)])).cuda()
        ref = eng.run(new).clone()
        ref_db = eng.db.clone()
        torch.cuda.synchronize()
        rf.copy_(new)
        got = g.replay()
        torch.cuda.synchronize()
        assert torch.equal(got, ref)
        assert torch.equal(eng.db, ref_db)
    eng.close()


@pytest.mark.parametrize("T", [1536, 1000, 4099])
def test_decomposition_odd_element_count_is_position_independent(T):
    """Odd element counts: the real-pair FFT pairs rows only within one
    (frame, transmit), so every frame of a batch equals its own single-frame
    decomposition bit for bit, whatever its position."""
    torch = _torch()
    arr = kb.TransducerArray(63, 0.3e-3, 5e6, 20e6, 0.6)
    params = kb.AcquisitionParams(C, np.linspace(-0.15, 0.15, 5), T)
    rx = kb.uniform_vernier_angles(5, 3, 0.15, 0)
    grid = kb.ImageGrid(-2e-3, 3e-3, 0.1e-3, 0.1e-3, 8, 8)
    frames = 3
    rf = torch.from_numpy(np.stack([configs.noise_rf(5, 63, T, seed=60 + f)
                                    for f in range(frames)])).cuda()
    eng = kb.KKEngine(arr, params, rx, grid, frames=frames, want_db=False)
    batch = eng.decompose(rf).clone()
    for f in range(frames):
        one = eng.decompose(rf[f:f + 1].contiguous(), n_frames=1).clone()
        torch.cuda.synchronize()
        assert torch.equal(one[0], batch[f]), f
    eng.close()
