"""The K5 instance bench.py times, pinned to the oracle.

bench.py's step gathers 400 config-4 frames per launch, which dispatches to
the 32 x 64-tile instance with two frames per CTA (KKB_KK_INST_BIG_FR).  A
63-frame batch reaches it through the normal dispatch, 16- and 11-frame
batches are forced onto it; the test asserts which instance ran (via
kkb_kk_last_instance), and the odd frame counts make the last CTA run the
one-frame tail.  Every frame is compared with
the oracle (reference kk on the oracle's own decomposition) and with a
single-frame launch of the same traces, which dispatches to the 16 x 16
instance: the per-pixel sums run in the same order, so they must agree bit
for bit.

Tolerances: IQ rel L2 <= 1e-5 per frame (north star); batch vs single
frame and instance vs instance: bit-exact.
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


@pytest.mark.parametrize("F,force", [(63, None), (16, "big_fr"), (11, "big_fr")])
def test_bench_instance_matches_oracle_every_frame(oracle, monkeypatch, F, force):
    """63 frames reach the two-frames-per-CTA instance through the default
    dispatch (odd: the last CTA runs the one-frame tail); 16 and 11 frames are
    forced onto it (KKB_KK_INST=big_fr)."""
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
    assert _lib.last_instance() == _lib.KKB_KK_INST_BIG_FR
    assert _lib.take_device_error() == 0
    # every frame again as a one-frame launch (16 x 16 instance): bit-identical
    P = g.nx * g.nz
    single = torch.empty_like(iq)
    for f in range(F):
        _lib.call("kkb_kk_plan_run", eng._kk, dev.ptr(eng.traces[f]), 1, 0, dev.ptr(single[f]),
                  _lib.KKB_OUT_C64, P, None, None, dev.stream_handle())
    torch.cuda.synchronize()
    assert _lib.last_instance() == _lib.KKB_KK_INST_SMALL
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


def test_dispatch_follows_the_wave_model():
    """The default dispatch (wave model, kk_gather.cu select_instance) on the
    measured shapes: bench workload -> two frames per CTA; one config-1 frame
    -> 16 x 16 tiles; one config-5 frame -> 32 x 64 tiles."""
    import torch

    for cfg, F, want in ((4, 400, _lib.KKB_KK_INST_BIG_FR), (1, 1, _lib.KKB_KK_INST_SMALL),
                         (5, 1, _lib.KKB_KK_INST_BIG)):
        w = configs.config4(frames=F) if cfg == 4 else configs.CONFIGS[cfg]()
        p, arr, rx, g = w.params, w.array, w.receive, w.grid
        eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False)
        eng.traces.zero_()
        eng.gather()
        torch.cuda.synchronize()
        assert _lib.last_instance() == want, (cfg, F, _lib.last_instance())
        eng.close()


def test_tensor_core_gather_experiment_matches_oracle(oracle, monkeypatch):
    """The opt-in tcgen05 gather (KKB_KK_INST=tc; slower than the FMA
    instances, kept as the measured experiment of DESIGN.md): a 32-frame
    config-4 batch within 1e-5 rel L2 of the oracle per frame, and each frame
    independent of the batch it is gathered in (rel 0 between a batch and
    single-frame tensor-core launches is not required: only the 1e-5 bound)."""
    import torch

    F = 32
    w = configs.config4(frames=F)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    fs, c = arr.sampling_frequency, p.sound_speed
    rf = _frames(w, F, 900)
    eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False)
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
        ref = oracle.kk_kernel(tr, *luts, np.ones(rx.num_angles), fs, shift)
        assert rel_l2(got[f], ref) <= 1e-5, f
    eng.close()
