"""The fused stage-1 -> tensor-core path bench.py times (KKEngine(fuse_tc=
True)): K3 writes the tensor-core gather's split fp16 planes directly
(kkb_decomposer_run_planes, per-frame scale from an L1 bound of the
contracted bins) and the gather reads them (kkb_kk_plan_run_planes), with no
complex64 traces in between.  Checked against the unfused engine (same
decomposition, traces -> frame max -> split -> gather), against the oracle
frame by frame, and for the NaN / Inf standby (K3 then writes the traces and
the FMA gather runs on them).

Tolerances: IQ rel L2 <= 1e-5 per frame vs the oracle (north star); fused vs
unfused: IQ <= 3e-6, |IQ|^2 <= 6e-6 per frame (different power-of-two scales
round the fp16 halves differently); NaN pattern bit-identical to the FMA
gather's.
"""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import _lib, configs  # noqa: E402


def _rf(w, F, seed0, distinct=8):
    import torch

    p, arr = w.params, w.array
    base = np.stack([configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=seed0 + d)
                     for d in range(min(distinct, F))])
    reps = (F + len(base) - 1) // len(base)
    return base, torch.from_numpy(base).cuda().repeat(reps, 1, 1, 1)[:F].contiguous()


def _rel(a, b):
    import torch

    return float((torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b)).item())


@pytest.mark.parametrize("F", [400, 100])
def test_fused_matches_unfused_and_oracle(oracle, F):
    import torch

    w = configs.config4(frames=F)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    base, rf = _rf(w, F, 300)
    fused = kb.KKEngine(arr, p, rx, g, frames=F, fuse_tc=True)
    plain = kb.KKEngine(arr, p, rx, g, frames=F)
    assert fused.fused and not plain.fused
    fused.decompose(rf)
    fused.gather()
    torch.cuda.synchronize()
    assert _lib.last_instance() == _lib.KKB_KK_INST_TC
    plain.decompose(rf)
    plain.gather()
    torch.cuda.synchronize()
    assert _lib.take_device_error() == 0
    for f in range(F):
        assert _rel(fused.iq[f], plain.iq[f]) <= 3e-6, f
        assert _rel(fused.inten[f], plain.inten[f]) <= 6e-6, f
    mf, mp = fused.fmax.view(torch.float32), plain.fmax.view(torch.float32)
    assert bool(((mf - mp).abs() <= 1e-5 * mp.abs()).all())
    # whole-path run() takes the fused route too
    fused.run(rf)
    torch.cuda.synchronize()
    got = fused.iq.cpu().numpy()
    fs, c = arr.sampling_frequency, p.sound_speed
    luts = oracle.kk_luts(g.x, g.z, p.transmit_angles, rx.angles, c)
    shift = (0.0 - p.start_time) * fs
    for f in (0, 63, F - 1):
        tr = oracle.decompose_f64(base[f % len(base)], fs, arr.positions, rx.angles, c)
        ref = oracle.kk_kernel(tr, *luts, np.ones(rx.num_angles), fs, shift)
        assert rel_l2(got[f], ref) <= 1e-5, f
    fused.close()
    plain.close()


def test_fused_nonfinite_standby(monkeypatch):
    import torch

    F = 64
    w = configs.config4(frames=F)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    _, rf = _rf(w, F, 500)
    rf[9, 2, 40, 333] = float("nan")
    fused = kb.KKEngine(arr, p, rx, g, frames=F, fuse_tc=True, want_db=False)
    plain = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False)
    fused.decompose(rf)
    fused.gather()
    monkeypatch.setenv("KKB_KK_TC", "0")
    plain.decompose(rf)
    plain.gather()
    torch.cuda.synchronize()
    monkeypatch.delenv("KKB_KK_TC")
    assert int(fused._nonfinite.item()) != 0
    assert torch.equal(torch.view_as_real(fused.traces).isnan(), torch.view_as_real(plain.traces).isnan())
    a, b = torch.view_as_real(fused.iq), torch.view_as_real(plain.iq)
    assert bool(b.isnan().any())
    assert torch.equal(a.isnan(), b.isnan())
    m = ~b.isnan()
    assert torch.equal(a[m], b[m])
    fused.close()
    plain.close()


@pytest.mark.parametrize("cfg", [2, 3])
def test_fused_other_lengths(oracle, cfg):
    """T = 2048 workloads (config 2: 15 x 5 pairs on 256 x 400 px; config 3's
    dense vernier set, 81 pairs on 384 x 512): the fused path against the
    unfused engine (every frame) and the oracle (first and last frame)."""
    import torch

    F = 56
    w = configs.CONFIGS[cfg]()
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    base, rf = _rf(w, F, 900 + cfg, distinct=4)
    fused = kb.KKEngine(arr, p, rx, g, frames=F, fuse_tc=True, want_db=False)
    plain = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False)
    assert fused.fused
    fused.run(rf)
    plain.run(rf)
    torch.cuda.synchronize()
    for f in range(F):
        assert _rel(fused.iq[f], plain.iq[f]) <= 3e-6, f
    got = fused.iq.cpu().numpy()
    fs, c = arr.sampling_frequency, p.sound_speed
    luts = oracle.kk_luts(g.x, g.z, p.transmit_angles, rx.angles, c)
    shift = (0.0 - p.start_time) * fs
    for f in (0, F - 1):
        tr = oracle.decompose_f64(base[f % len(base)], fs, arr.positions, rx.angles, c)
        ref = oracle.kk_kernel(tr, *luts, np.ones(rx.num_angles), fs, shift)
        assert rel_l2(got[f], ref) <= 1e-5, (cfg, f)
    fused.close()
    plain.close()


def test_fused_falls_back_when_ineligible():
    """Config 1's steep delays exceed the tensor-core tile's 32-sample
    windows: fuse_tc quietly keeps the complex64 path (and small batches, or
    batches below the crossover, never fuse)."""
    w = configs.config1()
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    assert not kb.KKEngine(arr, p, rx, g, frames=64, fuse_tc=True).fused
    w4 = configs.config4(frames=16)
    assert not kb.KKEngine(w4.array, w4.params, w4.receive, w4.grid, frames=16, fuse_tc=True).fused


@pytest.mark.parametrize("fuse", [True, False])
def test_tensor_core_path_graph_replay(fuse):
    """KKEngine.capture on a 64-frame config-4 batch (the tcgen05 gather, with
    and without the fused planes): replays on new RF equal the eager run bit
    for bit (the gather's scratch is stream-ordered, so it lives in the graph)."""
    import torch

    F = 64
    w = configs.config4(frames=F)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    eng = kb.KKEngine(arr, p, rx, g, frames=F, fuse_tc=fuse)
    _, rf0 = _rf(w, F, 40, distinct=2)
    rf = rf0.clone()
    graph = eng.capture(rf)
    for seed in (50, 60):
        _, new = _rf(w, F, seed, distinct=2)
        ref = eng.run(new).clone()
        torch.cuda.synchronize()
        assert _lib.last_instance() == _lib.KKB_KK_INST_TC
        rf.copy_(new)
        got = graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(got, ref)
    eng.close()
