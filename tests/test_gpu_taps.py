"""Tap exactness of the PRODUCTION gather (K5), every instance.

Index-encoding traces (oracle.tap_encoding): frame f holds nonzero data only
for one (transmit, receive) pair (n_f, m_f) — sample t = (t + 1) + i*h(t),
h a scrambled bijection — and the weights are ones, so each pixel of frame f
is exactly the tap K5 read for that pair: the lerp of samples i0, i0 + 1 at
the 23-bit fraction (linear), or sample j (nearest), or 0 out of window.
oracle.kk_tap_values computes that value from the reference's own tap index
and window rule (beamform.py:225-235), so a bit-exact image proves, for every
(pixel, pair), the index, the in-window predicate and the staged-window
addressing (per-frame window blocks of the two-frames-per-CTA instance, the
odd-frame tail, the clamp at the window end) of the kernel that runs in the
benchmark — not of the kk_taps diagnostic twin.  One frame per pair puts all
N*M pairs in one batched launch.  Every plan also proves at creation
(kk_check_windows: every (pixel, pair) through the gather's own index
arithmetic against each tile size's staged window) that no tap can be
clamped at its window's end: kkb_kk_plan_window_check must be 0 and the
device error word (KKB_DEVERR_KK_WINDOW) clear; a fault-injection test shows
the proof catching undersized windows and the dispatch routing around them.

The tensor-core gather (kk_gather_tc.cu; the default for linear batches of
>= 48 frames, so "natural" below for linear) multiplies split-fp16 weights
and samples: its taps are checked to 2e-6 relative per pixel instead, which
still pins every index and in-window decision (a wrong sample or a missed
rejection is off by >= 1 in value, ~5e-4 relative).

Tolerance: bit-exact (torch.equal / np.array_equal) for the FMA instances;
2e-6 relative per pixel for the tensor-core gather.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2603_22496_b200 import _device as dev  # noqa: E402
from paper_2603_22496_b200 import _lib, configs  # noqa: E402

INSTANCES = ["natural", "big_fr", "big", "mid", "small", "direct", "tc"]
CODE = {"big_fr": _lib.KKB_KK_INST_BIG_FR, "big": _lib.KKB_KK_INST_BIG, "mid": _lib.KKB_KK_INST_MID,
        "small": _lib.KKB_KK_INST_SMALL, "direct": _lib.KKB_KK_INST_DIRECT, "tc": _lib.KKB_KK_INST_TC}


def _assert_taps(out, ref, code, what):
    if code == _lib.KKB_KK_INST_TC:  # split-fp16 products: per-pixel relative bound
        err = (out - ref).abs()
        assert bool((err <= 2e-6 * ref.abs()).all()), (what, float(err.max()))
    else:
        bad = out != ref
        assert not bool(bad.any()), (what, int(bad.sum()))


def _plan(luts, N, M, T, nx, nz, fs, shift, linear):
    d = [dev.to_device(np.ascontiguousarray(a)) for a in luts]
    kp = ctypes.c_void_p()
    _lib.call("kkb_kk_plan_create", *[x.data_ptr() for x in d], N, M, T, nx, nz, None, float(fs),
              float(shift), int(linear), dev.stream_handle(), ctypes.byref(kp))
    return kp, d


def _encoded(pairs, N, M, T):
    import torch

    from oracle import kkbeam_oracle as O

    F = len(pairs)
    data = torch.zeros((F, N, M, T), dtype=torch.complex64, device="cuda")
    enc = torch.from_numpy(O.tap_encoding(T).astype(np.complex64)).cuda()
    n_idx = torch.tensor([p[0] for p in pairs], device="cuda")
    m_idx = torch.tensor([p[1] for p in pairs], device="cuda")
    data[torch.arange(F, device="cuda"), n_idx, m_idx] = enc
    return data


def _run(kp, data, nx, nz, monkeypatch, inst):
    import torch

    if inst == "natural":
        monkeypatch.delenv("KKB_KK_INST", raising=False)
    else:
        monkeypatch.setenv("KKB_KK_INST", inst)
    F, N, M, T = data.shape
    out = torch.empty((F, nx, nz), dtype=torch.complex64, device="cuda")
    _lib.call("kkb_kk_plan_run", kp, dev.ptr(data), F, N * M * T, dev.ptr(out), _lib.KKB_OUT_C64,
              nx * nz, None, None, dev.stream_handle())
    torch.cuda.synchronize()
    got_inst = _lib.last_instance()
    assert _lib.take_device_error() == 0, "a tap index was clamped at the staged window's end"
    monkeypatch.delenv("KKB_KK_INST", raising=False)
    return out, got_inst


def _luts(oracle, w):
    g, p, rx = w.grid, w.params, w.receive
    return oracle.kk_luts(g.x, g.z, p.transmit_angles, rx.angles, p.sound_speed)


@pytest.mark.parametrize("linear", [True, False])
@pytest.mark.parametrize("cfg", [1, 4])
def test_production_gather_taps_bit_exact(oracle, monkeypatch, cfg, linear):
    """Configs 1 and 4: all N*M = 121 pairs as 121 frames in one launch
    (odd frame count: the FR = 2 instance's tail), every instance."""
    import torch

    w = configs.config1() if cfg == 1 else configs.config4(frames=1)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    N, M, T, fs = p.num_transmits, rx.num_angles, p.num_samples, arr.sampling_frequency
    shift = (0.0 - p.start_time) * fs
    luts = _luts(oracle, w)
    exp = oracle.kk_tap_values(*luts, fs, shift, T, linear)      # (X, Z, N, M)
    pairs = [(n, m) for n in range(N) for m in range(M)]
    ref = torch.from_numpy(np.ascontiguousarray(np.moveaxis(exp.reshape(g.nx, g.nz, N * M), -1, 0)))
    data = _encoded(pairs, N, M, T)
    kp, keep = _plan(luts, N, M, T, g.nx, g.nz, fs, shift, linear)
    assert _lib.load().kkb_kk_plan_window_check(kp) == 0   # every tile size proven at plan time
    try:
        for inst in INSTANCES:
            out, code = _run(kp, data, g.nx, g.nz, monkeypatch, inst)
            if inst == "tc" and cfg == 1:
                assert code != _lib.KKB_KK_INST_TC  # too steep for its 4 x 32 tile: not eligible
                continue
            if inst != "natural":
                assert code == CODE[inst], (inst, code)
            _assert_taps(out.cpu(), ref, code, (cfg, linear, inst))
    finally:
        _lib.load().kkb_kk_plan_destroy(kp)


def test_production_gather_taps_multiset(oracle, monkeypatch):
    """The one-launch multi-set form (kkb_kk_plan_run_sets, three receive
    sets) on config 4's index-encoded pairs: set j's image is the tap value
    when m_f lies in set j, else 0; intensity = |tap|^2."""
    import torch

    w = configs.config4(frames=1)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    N, M, T, fs = p.num_transmits, rx.num_angles, p.num_samples, arr.sampling_frequency
    shift = (0.0 - p.start_time) * fs
    luts = _luts(oracle, w)
    exp = oracle.kk_tap_values(*luts, fs, shift, T, True)
    pairs = [(n, m) for n in range(N) for m in range(M)]
    F, P = len(pairs), g.nx * g.nz
    data = _encoded(pairs, N, M, T)
    bounds = [0, 4, 7, M]
    kp, keep = _plan(luts, N, M, T, g.nx, g.nz, fs, shift, True)
    try:
        for inst in ("natural", "small", "direct"):
            if inst != "natural":
                monkeypatch.setenv("KKB_KK_INST", inst)
            iq = torch.empty((3, F, g.nx, g.nz), dtype=torch.complex64, device="cuda")
            inten = torch.empty((F, g.nx, g.nz), dtype=torch.float32, device="cuda")
            b = (ctypes.c_int * 4)(*bounds)
            _lib.call("kkb_kk_plan_run_sets", kp, dev.ptr(data), F, N * M * T, 3, b, dev.ptr(iq),
                      _lib.KKB_OUT_C64, P, F * P, dev.ptr(inten), None, 0, dev.stream_handle())
            torch.cuda.synchronize()
            code = _lib.last_instance()
            monkeypatch.delenv("KKB_KK_INST", raising=False)
            assert code & _lib.KKB_KK_INST_SETS
            assert _lib.take_device_error() == 0
            iq_h = iq.cpu().numpy()
            for f, (n, m) in enumerate(pairs):
                j = int(np.searchsorted(bounds, m, side="right") - 1)
                for s in range(3):
                    e = exp[:, :, n, m] if s == j else np.zeros((g.nx, g.nz), np.complex64)
                    assert np.array_equal(iq_h[s, f], e), (inst, f, s)
            v = exp.reshape(P, N * M).T
            ref_i = (v.real.astype(np.float32) * v.real.astype(np.float32)
                     + v.imag.astype(np.float32) * v.imag.astype(np.float32))
            assert np.allclose(inten.cpu().numpy().reshape(F, P), ref_i, rtol=1e-6, atol=0)
    finally:
        _lib.load().kkb_kk_plan_destroy(kp)


@pytest.mark.parametrize("linear", [True, False])
def test_production_gather_taps_config5_row_block(oracle, monkeypatch, linear):
    """Config 5 (31 x 31 pairs, T = 4096): a 32-row block of the 1024 x 2048
    image (one rank's share at 32 GPUs, the RowBlockKK table slice), all 961
    pairs — one launch of 31 frames per transmit — through the instance the
    block dispatches to, the mid / small tiles and the per-pixel kernel."""
    import torch

    w = configs.config5()
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    N, M, T, fs = p.num_transmits, rx.num_angles, p.num_samples, arr.sampling_frequency
    shift = (0.0 - p.start_time) * fs
    ltx, ltz, lrx, lrz = _luts(oracle, w)
    r0, r1 = 480, 512
    luts = (ltx[r0:r1], ltz, lrx[r0:r1], lrz)
    nx, nz = r1 - r0, g.nz
    kp, keep = _plan(luts, N, M, T, nx, nz, fs, shift, linear)
    try:
        for n in range(N):
            exp = oracle.kk_tap_values(luts[0][:, n:n + 1], ltz[:, n:n + 1], luts[2], lrz, fs, shift, T,
                                       linear)[:, :, 0, :]                    # (nx, nz, M)
            ref = torch.from_numpy(np.ascontiguousarray(np.moveaxis(exp, -1, 0)))
            data = _encoded([(n, m) for m in range(M)], N, M, T)
            for inst in (["natural", "mid", "small", "direct"] if n % 10 == 0 else ["natural"]):
                out, code = _run(kp, data, nx, nz, monkeypatch, inst)
                if inst != "natural":
                    assert code == CODE[inst], (inst, code)
                bad = out.cpu() != ref
                assert not bool(bad.any()), (n, linear, inst, int(bad.sum()))
            del data
    finally:
        _lib.load().kkb_kk_plan_destroy(kp)


def test_window_proof_catches_undersized_windows(oracle, monkeypatch):
    """Fault injection: KKB_KK_WINDOW_SHRINK makes every staged window too
    short.  The plan-time proof must flag the tile sizes whose taps would be
    clamped (and raise the device error word), the dispatch must then avoid
    them, and the image must stay identical to the correctly sized plan's."""
    import torch

    monkeypatch.setenv("KKB_KK_TC", "0")  # the subject is the FMA instances' staged windows
    w = configs.config4(frames=1)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    N, M, T, fs = p.num_transmits, rx.num_angles, p.num_samples, arr.sampling_frequency
    shift = (0.0 - p.start_time) * fs
    luts = _luts(oracle, w)
    pairs = [(n, m) for n in range(N) for m in range(M)]
    data = _encoded(pairs, N, M, T)
    good, keep_g = _plan(luts, N, M, T, g.nx, g.nz, fs, shift, True)
    assert _lib.take_device_error() == 0
    ref, _ = _run(good, data, g.nx, g.nz, monkeypatch, "natural")
    monkeypatch.setenv("KKB_KK_WINDOW_SHRINK", "6")
    bad, keep_b = _plan(luts, N, M, T, g.nx, g.nz, fs, shift, True)
    monkeypatch.delenv("KKB_KK_WINDOW_SHRINK")
    flags = _lib.load().kkb_kk_plan_window_check(bad)
    assert flags != 0
    assert _lib.take_device_error() & _lib.KKB_DEVERR_KK_WINDOW
    for inst in INSTANCES[:-1]:   # the FMA instances (the tensor-core windows are exact per tile)
        out, code = _run(bad, data, g.nx, g.nz, monkeypatch, inst)
        assert not (flags & (1 << code)), (inst, code, flags)   # a flagged instance never runs
        assert torch.equal(out, ref), inst
    for kp in (good, bad):
        _lib.load().kkb_kk_plan_destroy(kp)
