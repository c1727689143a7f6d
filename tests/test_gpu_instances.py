"""The K5 instances bench.py times, pinned to the oracle.

bench.py's step gathers 400 config-4 frames per launch; linear batches of
>= 48 frames dispatch to the tensor-core gather (KKB_KK_INST_TC,
kk_gather_tc.cu), smaller ones to the FMA instances (wave model).  A
63-frame batch reaches the tensor-core gather through the normal dispatch
and the two-frames-per-CTA FMA instance (KKB_KK_INST_BIG_FR) when forced, as
do 16- and 11-frame batches; the test asserts which instance ran (via
kkb_kk_last_instance), and the odd frame counts make the last CTA run the
one-frame tail.  Every frame is compared with the oracle (reference kk on
the oracle's own decomposition) and with a single-frame launch of the same
traces through the same kind of gather (16 x 16 FMA instance, or the
tensor-core gather forced): a pixel's sum runs in the same order whatever
the batch, so they must agree bit for bit.  The tensor-core gather's NaN /
Inf standby (the FMA gather runs instead) and its intensity / frame-max
epilogue are covered too.

Tolerances: IQ rel L2 <= 1e-5 per frame (north star); batch vs single
frame and FMA instance vs FMA instance: bit-exact; tensor-core vs FMA
gather: IQ rel L2 <= 3e-6 per frame (split-fp16 products, measured ~9e-7),
|IQ|^2 <= 6e-6 (twice the relative error of IQ).
"""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import _device as dev  # noqa: E402
from paper_2603_22496_b200 import _lib, configs  # noqa: E402


def _frames(w, F, seed0):
    p, arr = w.params, w.array
    return np.stack([configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=seed0 + f)
                     for f in range(F)])


@pytest.mark.parametrize("F,force,want", [(63, None, _lib.KKB_KK_INST_TC), (63, "big_fr", _lib.KKB_KK_INST_BIG_FR),
                                          (16, "big_fr", _lib.KKB_KK_INST_BIG_FR),
                                          (11, "big_fr", _lib.KKB_KK_INST_BIG_FR)])
def test_bench_instance_matches_oracle_every_frame(oracle, monkeypatch, F, force, want):
    """63 frames reach the tensor-core gather through the default dispatch;
    63, 16 and 11 frames forced onto the two-frames-per-CTA FMA instance
    (odd: the last CTA runs the one-frame tail)."""
    import torch

    w = configs.config4(frames=F)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    fs, c = arr.sampling_frequency, p.sound_speed
    rf = _frames(w, F, 700)
    eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False)
    if force:
        monkeypatch.setenv("KKB_KK_INST", force)
    iq = eng.run(torch.from_numpy(rf).cuda()).clone()
    torch.cuda.synchronize()
    monkeypatch.delenv("KKB_KK_INST", raising=False)
    assert _lib.last_instance() == want
    assert _lib.take_device_error() == 0
    # every frame again as a one-frame launch of the same kind of gather
    tc = want == _lib.KKB_KK_INST_TC
    if tc:
        monkeypatch.setenv("KKB_KK_INST", "tc")
    P = g.nx * g.nz
    single = torch.empty_like(iq)
    for f in range(F):
        _lib.call("kkb_kk_plan_run", eng._kk, dev.ptr(eng.traces[f]), 1, 0, dev.ptr(single[f]),
                  _lib.KKB_OUT_C64, P, None, None, dev.stream_handle())
    torch.cuda.synchronize()
    monkeypatch.delenv("KKB_KK_INST", raising=False)
    assert _lib.last_instance() == (_lib.KKB_KK_INST_TC if tc else _lib.KKB_KK_INST_SMALL)
    assert torch.equal(iq, single)
    # every frame against the oracle: reference kk on the oracle's decomposition
    luts = oracle.kk_luts(g.x, g.z, p.transmit_angles, rx.angles, c)
    shift = (0.0 - p.start_time) * fs
    got = iq.cpu().numpy()
    for f in range(F):
        tr = oracle.decompose_f64(rf[f], fs, arr.positions, rx.angles, c)
        ref = oracle.kk_kernel(tr, *luts, np.ones(rx.num_angles), fs, shift)
        e = rel_l2(got[f], ref)
        assert e <= 1e-5, (F, f, e)
    eng.close()


def test_every_instance_bit_identical(monkeypatch):
    """One 6-frame config-4 batch through all five K5 instances (forced with
    KKB_KK_INST; each asserted by kkb_kk_last_instance): identical images."""
    import torch

    w = configs.config4(frames=6)
    p, arr, g = w.params, w.array, w.grid
    rf = _frames(w, 6, 30)
    eng = kb.KKEngine(arr, p, w.receive, g, frames=6, want_db=False)
    eng.decompose(torch.from_numpy(rf).cuda())
    outs = {}
    for name, code in (("big_fr", _lib.KKB_KK_INST_BIG_FR), ("big", _lib.KKB_KK_INST_BIG),
                       ("mid", _lib.KKB_KK_INST_MID), ("small", _lib.KKB_KK_INST_SMALL),
                       ("direct", _lib.KKB_KK_INST_DIRECT)):
        monkeypatch.setenv("KKB_KK_INST", name)
        eng.gather()
        torch.cuda.synchronize()
        assert _lib.last_instance() == code, name
        outs[name] = (eng.iq.clone(), eng.inten.clone(), eng.fmax.clone())
    monkeypatch.delenv("KKB_KK_INST")
    assert _lib.take_device_error() == 0
    ref = outs["big_fr"]
    for name, o in outs.items():
        for a, b in zip(o, ref):
            assert torch.equal(a, b), name
    eng.close()


def test_dispatch_follows_the_wave_model(monkeypatch):
    """The default dispatch on the measured shapes: the bench workload (400
    linear frames) -> the tensor-core gather, or with KKB_KK_TC=0 the wave
    model's choice (kk_gather.cu select_instance), two frames per CTA; one
    config-1 frame -> 16 x 16 tiles; one config-5 frame -> 32 x 64 tiles."""
    import torch

    for cfg, F, tc, want in ((4, 400, True, _lib.KKB_KK_INST_TC), (4, 400, False, _lib.KKB_KK_INST_BIG_FR),
                             (1, 1, True, _lib.KKB_KK_INST_SMALL), (5, 1, True, _lib.KKB_KK_INST_BIG)):
        if not tc:
            monkeypatch.setenv("KKB_KK_TC", "0")
        w = configs.config4(frames=F) if cfg == 4 else configs.CONFIGS[cfg]()
        p, arr, rx, g = w.params, w.array, w.receive, w.grid
        eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False)
        eng.traces.zero_()
        eng.gather()
        torch.cuda.synchronize()
        monkeypatch.delenv("KKB_KK_TC", raising=False)
        assert _lib.last_instance() == want, (cfg, F, _lib.last_instance())
        eng.close()


@pytest.mark.parametrize("linear", [True, False])
def test_tensor_core_gather_matches_oracle(oracle, monkeypatch, linear):
    """The tcgen05 gather forced on a 32-frame config-4 batch (below the
    default crossover), linear and nearest: within 1e-5 rel L2 of the
    oracle per frame."""
    import torch

    F = 32
    w = configs.config4(frames=F)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    fs, c = arr.sampling_frequency, p.sound_speed
    rf = _frames(w, F, 900)
    eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False, interpolation="linear" if linear else "nearest")
    eng.decompose(torch.from_numpy(rf).cuda())
    monkeypatch.setenv("KKB_KK_INST", "tc")
    eng.gather()
    torch.cuda.synchronize()
    monkeypatch.delenv("KKB_KK_INST")
    assert _lib.last_instance() == _lib.KKB_KK_INST_TC
    assert _lib.take_device_error() == 0
    got = eng.iq.cpu().numpy()
    luts = oracle.kk_luts(g.x, g.z, p.transmit_angles, rx.angles, c)
    shift = (0.0 - p.start_time) * fs
    for f in (0, 7, 31):
        tr = oracle.decompose_f64(rf[f], fs, arr.positions, rx.angles, c)
        ref = oracle.kk_kernel(tr, *luts, np.ones(rx.num_angles), fs, shift, linear=linear)
        assert rel_l2(got[f], ref) <= 1e-5, f
    eng.close()


def test_tensor_core_epilogue_matches_fma(monkeypatch):
    """Intensity |IQ|^2 and the per-frame max (the dB path's inputs) from the
    tensor-core gather against the FMA gather on a 100-frame batch (a 36-frame
    tail block): IQ rel L2 <= 3e-6 and intensity <= 6e-6 per frame, frame max
    within 1e-5."""
    import torch

    F = 100
    w = configs.config4(frames=F)
    p, arr, g = w.params, w.array, w.grid
    rf = _frames(w, F, 1200)
    eng = kb.KKEngine(arr, p, w.receive, g, frames=F, want_db=True)
    eng.decompose(torch.from_numpy(rf).cuda())
    outs = {}
    for tc in ("1", "0"):
        monkeypatch.setenv("KKB_KK_TC", tc)
        eng.gather()
        torch.cuda.synchronize()
        outs[tc] = (_lib.last_instance(), eng.iq.clone(), eng.inten.clone(),
                    eng.fmax.clone().view(torch.float32))
    monkeypatch.delenv("KKB_KK_TC")
    assert outs["1"][0] == _lib.KKB_KK_INST_TC and outs["0"][0] == _lib.KKB_KK_INST_BIG_FR
    for a, b, tol in zip(outs["1"][1:3], outs["0"][1:3], (3e-6, 6e-6)):
        for f in range(F):
            e = float((torch.linalg.vector_norm(a[f] - b[f]) / torch.linalg.vector_norm(b[f])).item())
            assert e <= tol, (f, e, tol)
    ft, ff = outs["1"][3], outs["0"][3]
    assert bool(((ft - ff).abs() <= 1e-5 * ff.abs()).all())


def test_tensor_core_nonfinite_standby(monkeypatch):
    """A NaN and an Inf sample in a 64-frame batch: the tensor-core gather
    stands down on the device and the FMA standby computes the batch, so the
    image (NaN / Inf pattern included) is bit-identical to the FMA gather's,
    where the reference spreads a non-finite sample only to the pixels that
    tap it."""
    import torch

    F = 64
    w = configs.config4(frames=F)
    p, arr, g = w.params, w.array, w.grid
    rf = _frames(w, F, 1500)
    eng = kb.KKEngine(arr, p, w.receive, g, frames=F, want_db=False)
    eng.decompose(torch.from_numpy(rf).cuda())
    eng.traces[5, 3, 4, 700] = float("nan")
    eng.traces[40, 0, 10, 300] = complex(float("inf"), 0.0)
    outs = {}
    for tc in ("1", "0"):
        monkeypatch.setenv("KKB_KK_TC", tc)
        eng.gather()
        torch.cuda.synchronize()
        outs[tc] = (_lib.last_instance(), eng.iq.clone())
    monkeypatch.delenv("KKB_KK_TC")
    assert outs["1"][0] == _lib.KKB_KK_INST_TC
    a, b = outs["1"][1], outs["0"][1]
    assert bool(torch.isnan(b.real).any() | torch.isnan(b.imag).any())
    va, vb = torch.view_as_real(a), torch.view_as_real(b)
    assert torch.equal(torch.isnan(va), torch.isnan(vb))
    m = ~torch.isnan(vb)
    assert torch.equal(va[m], vb[m])
    eng.close()


def test_bench_workload_tensor_core_gather(oracle, monkeypatch):
    """The exact configuration bench.py times: 400 config-4 frames in one
    launch (seven 64-frame blocks, the last of 2 frame groups), through the
    default dispatch -> the tensor-core gather.  Every frame against the
    oracle-pinned FMA gather (KKB_KK_TC=0 -> big_fr), sampled frames against
    the oracle itself, and repeated input frames (8 distinct frames tiled, as
    in bench.py) bit-identical wherever they sit in the batch."""
    import torch

    F, D = 400, 8
    w = configs.config4(frames=F)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    fs, c = arr.sampling_frequency, p.sound_speed
    base = _frames(w, D, 2000)
    eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=True)
    rf = torch.from_numpy(base).cuda().repeat(F // D, 1, 1, 1)
    eng.decompose(rf)
    del rf
    outs = {}
    for tc in ("1", "0"):
        monkeypatch.setenv("KKB_KK_TC", tc)
        eng.gather()
        torch.cuda.synchronize()
        outs[tc] = (_lib.last_instance(), eng.iq.clone())
    monkeypatch.delenv("KKB_KK_TC")
    assert outs["1"][0] == _lib.KKB_KK_INST_TC and outs["0"][0] == _lib.KKB_KK_INST_BIG_FR
    assert _lib.take_device_error() == 0
    a, b = outs["1"][1], outs["0"][1]
    for f in range(F):
        e = float((torch.linalg.vector_norm(a[f] - b[f]) / torch.linalg.vector_norm(b[f])).item())
        assert e <= 3e-6, (f, e)
    for f in range(D, F):
        assert torch.equal(a[f], a[f % D]), f
    luts = oracle.kk_luts(g.x, g.z, p.transmit_angles, rx.angles, c)
    shift = (0.0 - p.start_time) * fs
    got = a.cpu().numpy()
    for f in (0, 63, 64, 383, 384, 399):
        tr = oracle.decompose_f64(base[f % D], fs, arr.positions, rx.angles, c)
        ref = oracle.kk_kernel(tr, *luts, np.ones(rx.num_angles), fs, shift)
        assert rel_l2(got[f], ref) <= 1e-5, f
    eng.close()
