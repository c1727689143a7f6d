"""The fused stage-1 kernel (K1 real FFT + K2 symmetric contraction in one
kernel, csrc/stage1_fused.cu) against the oracle and the three-kernel path.

Replaces rfft * one_sided / T (spectral.py:84-93) and the compress einsum
(compress.py:78-81).  Tolerances: decomposed traces rel L2 <= 1e-5 vs the
float64 oracle (north star) and <= 2e-6 vs the unfused K1 -> K2 path (the
fused kernel anchors its phase factors every four element pairs in float64
and steps them by the per-element rotation; the unfused path reads them from
a complex64 table: both round at the 1e-7 level).
"""

import ctypes

import numpy as np
import pytest

from conftest import C, DEG, rel_l2

pytestmark = pytest.mark.gpu

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import _lib, configs  # noqa: E402


def _traces(w, rf, fused):
    import torch

    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    eng = kb.KKEngine(arr, p, rx, g, frames=rf.shape[0], want_db=False)
    lib = _lib.load()
    assert lib.kkb_decomposer_fused(eng._dec) == 0   # opt-in
    _lib.call("kkb_decomposer_set_fused", eng._dec, int(fused))
    assert lib.kkb_decomposer_fused(eng._dec) == int(fused)
    tr = eng.decompose(torch.from_numpy(rf).cuda()).cpu().numpy()
    eng.close()
    return tr


def _workload(L, n_rx, T=1536, n_tx=11):
    arr = kb.TransducerArray(L, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    params = kb.AcquisitionParams(C, np.linspace(-10 * DEG, 10 * DEG, n_tx), T)
    rx = kb.uniform_vernier_angles(n_tx, n_rx, 10 * DEG, 1)
    grid = kb.ImageGrid(-2e-3, 5e-3, 0.1e-3, 0.1e-3, 8, 8)
    return configs.Workload(f"s1f_L{L}_M{n_rx}", arr, params, rx, grid)


def test_fused_at_config4_matches_oracle(oracle):
    F = 3
    w = configs.config4(frames=F)
    arr, p, rx = w.array, w.params, w.receive
    rf = np.stack([configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=80 + f)
                   for f in range(F)])
    fused = _traces(w, rf, True)
    plain = _traces(w, rf, False)
    assert rel_l2(fused, plain) <= 2e-6
    for f in range(F):
        ref = oracle.decompose_f64(rf[f], arr.sampling_frequency, arr.positions, rx.angles, p.sound_speed)
        assert rel_l2(fused[f], ref) <= 1e-5, f
        # every (transmit, receive) row on its own, not only the frame aggregate
        err = np.linalg.norm(fused[f] - ref, axis=-1) / np.linalg.norm(ref, axis=-1)
        assert err.max() <= 1e-5, (f, err.max())


@pytest.mark.parametrize("L,n_rx", [(64, 11), (128, 4), (256, 7), (8, 3)])
def test_fused_geometries_match_oracle(oracle, L, n_rx):
    """Element counts from one round (L = 8) to 32 rounds (L = 256), class
    counts with and without the theta = 0 receive angle."""
    w = _workload(L, n_rx)
    arr, p, rx = w.array, w.params, w.receive
    rf = np.stack([configs.noise_rf(p.num_transmits, L, p.num_samples, seed=90 + f) for f in range(2)])
    fused = _traces(w, rf, True)
    plain = _traces(w, rf, False)
    assert rel_l2(fused, plain) <= 2e-6
    ref = oracle.decompose_f64(rf[1], arr.sampling_frequency, arr.positions, rx.angles, C)
    assert rel_l2(fused[1], ref) <= 1e-5


def test_fused_dc_nyquist_and_point_echo(oracle):
    """Energy only in the DC and Nyquist bins (the bins the split assigns to
    special owners) and a single echo on one element."""
    w = configs.config4(frames=1)
    arr, p, rx = w.array, w.params, w.receive
    N, L, T = p.num_transmits, arr.num_elements, p.num_samples
    t = np.arange(T)
    rf = np.zeros((3, N, L, T), np.float32)
    rf[0] = 0.25                                   # DC only
    rf[1] = np.where(t % 2 == 0, 1.0, -1.0)        # Nyquist only
    rf[2, 3, 17, 700] = 1.0                        # one echo
    fused = _traces(w, rf, True)
    for f in range(3):
        ref = oracle.decompose_f64(rf[f], arr.sampling_frequency, arr.positions, rx.angles, p.sound_speed)
        assert rel_l2(fused[f], ref) <= 1e-5, f


def test_fused_int16_equals_float():
    import torch

    w = configs.config4(frames=2)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    q = np.random.default_rng(5).integers(-2000, 2000, size=(2, p.num_transmits, arr.num_elements,
                                                             p.num_samples)).astype(np.int16)
    eng = kb.KKEngine(arr, p, rx, g, frames=2, want_db=False)
    _lib.call("kkb_decomposer_set_fused", eng._dec, 1)
    assert _lib.load().kkb_decomposer_fused(eng._dec) == 1
    a = eng.decompose(torch.from_numpy(q).cuda()).cpu().numpy()
    b = eng.decompose(torch.from_numpy(q.astype(np.float32)).cuda()).cpu().numpy()
    eng.close()
    assert np.array_equal(a, b)


def test_fused_ineligible_plans():
    lib = _lib.load()
    # non-uniform array: the phase is not linear in the element index
    arr = kb.TransducerArray(16, 0.3e-3, 5e6, 20e6, 0.6)
    pos = arr.positions.copy()
    pos[3] += 1e-5
    pos[-4] -= 1e-5
    ang = np.array([-0.05, 0.0, 0.05])
    for positions, T in ((pos, 1536), (arr.positions, 1024)):
        h = ctypes.c_void_p()
        _lib.call("kkb_decomposer_create", 2, 16, T, np.ascontiguousarray(positions).ctypes.data,
                  ang.ctypes.data, 3, 20e6, C, 1, ctypes.byref(h))
        try:
            assert lib.kkb_decomposer_symmetric_classes(h) == 2
            assert lib.kkb_decomposer_fused(h) == 0
            with pytest.raises(kb.KKBeamError):
                _lib.call("kkb_decomposer_set_fused", h, 1)
        finally:
            lib.kkb_decomposer_destroy(h)
    # the uniform T = 1536 plan is eligible (opt-in) and switches both ways
    h = ctypes.c_void_p()
    _lib.call("kkb_decomposer_create", 2, 16, 1536, arr.positions.ctypes.data, ang.ctypes.data, 3, 20e6, C, 1,
              ctypes.byref(h))
    try:
        assert lib.kkb_decomposer_fused(h) == 0
        _lib.call("kkb_decomposer_set_fused", h, 1)
        assert lib.kkb_decomposer_fused(h) == 1
        _lib.call("kkb_decomposer_set_fused", h, 0)
        assert lib.kkb_decomposer_fused(h) == 0
    finally:
        lib.kkb_decomposer_destroy(h)


def test_engine_option_whole_path(oracle):
    """KKEngine(fused_stage1=True): the whole path (decomposition, gather,
    detection) against the default engine and the oracle's image."""
    import torch

    F = 2
    w = configs.config4(frames=F)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    rf = np.stack([configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=110 + f)
                   for f in range(F)])
    outs = []
    for fused in (True, False):
        eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False, fused_stage1=fused)
        assert _lib.load().kkb_decomposer_fused(eng._dec) == int(fused)
        outs.append(eng.run(torch.from_numpy(rf).cuda()).cpu().numpy().copy())
        eng.close()
    assert rel_l2(outs[0], outs[1]) <= 2e-6
    ref_tr = oracle.decompose_f64(rf[1], arr.sampling_frequency, arr.positions, rx.angles, p.sound_speed)
    luts = oracle.kk_luts(g.x, g.z, p.transmit_angles, rx.angles, p.sound_speed)
    shift = oracle.kk_resolved_shift(0.0, p.start_time, arr.sampling_frequency)
    ref = oracle.kk_kernel(ref_tr, *luts, np.ones(rx.num_angles), arr.sampling_frequency, shift)
    assert rel_l2(outs[0][1].reshape(ref.shape), ref) <= 1e-5


def test_engine_option_rejects_ineligible():
    arr = kb.TransducerArray(16, 0.3e-3, 5e6, 20e6, 0.6)
    params = kb.AcquisitionParams(C, np.linspace(-0.1, 0.1, 3), 1024)     # T != 1536
    rx = kb.uniform_vernier_angles(3, 3, 0.1, 1)
    grid = kb.ImageGrid(-1e-3, 2e-3, 0.1e-3, 0.1e-3, 4, 4)
    with pytest.raises(kb.ConfigError):
        kb.KKEngine(arr, params, rx, grid, frames=1, fused_stage1=True)


def test_fused_random_geometries(oracle):
    """Seeded random eligible geometries: element counts (multiples of 8),
    receive sets, pitches and sampling rates."""
    rng = np.random.default_rng(2026)
    for case in range(6):
        L = int(rng.integers(1, 33)) * 8
        n_tx = int(rng.integers(3, 12))
        n_rx = int(rng.integers(1, 12))
        fs = float(rng.uniform(16e6, 40e6))
        arr = kb.TransducerArray(L, float(rng.uniform(0.1e-3, 0.4e-3)), fs / 5, fs, 0.5)
        params = kb.AcquisitionParams(C, np.linspace(-12 * DEG, 12 * DEG, n_tx), 1536)
        rx = kb.uniform_vernier_angles(n_tx, n_rx, 12 * DEG, int(rng.integers(0, n_tx // 2 + 1)))
        grid = kb.ImageGrid(-2e-3, 5e-3, 0.1e-3, 0.1e-3, 8, 8)
        w = configs.Workload(f"rand{case}", arr, params, rx, grid)
        rf = configs.noise_rf(n_tx, L, 1536, seed=200 + case)[None]
        fused = _traces(w, rf, True)
        plain = _traces(w, rf, False)
        assert rel_l2(fused, plain) <= 2e-6, (case, L, n_rx)
        ref = oracle.decompose_f64(rf[0], fs, arr.positions, rx.angles, C)
        assert rel_l2(fused[0], ref) <= 1e-5, (case, L, n_rx)
