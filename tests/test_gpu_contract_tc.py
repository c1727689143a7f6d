"""The tensor-core (tcgen05, 3xTF32) form of the K2 contraction (north star:
"complex fp32 via split real GEMM or fp32 FMA, whichever ncu shows faster")
against the oracle and the FMA form.

Tolerances: decomposed traces rel L2 <= 1e-5 vs the oracle (north star; the
split-precision GEMM keeps fp32-level accuracy, so the 1e-3 TF32 allowance
is not used) and <= 5e-6 vs the FMA form (1.8e-6 at config 5's 256
elements: different fp32 summation orders).
"""

import numpy as np
import pytest

from conftest import C, DEG, rel_l2

pytestmark = pytest.mark.gpu

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import _lib, configs  # noqa: E402


def _traces(w, rf, tensor):
    import torch

    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    eng = kb.KKEngine(arr, p, rx, g, frames=rf.shape[0], want_db=False)
    if tensor:
        _lib.call("kkb_decomposer_set_contraction", eng._dec, _lib.KKB_CONTRACT_TENSOR)
        assert _lib.load().kkb_decomposer_contraction(eng._dec) == _lib.KKB_CONTRACT_TENSOR
    tr = eng.decompose(torch.from_numpy(rf).cuda()).cpu().numpy()
    eng.close()
    return tr


@pytest.mark.parametrize("cfg,F", [(1, 1), (4, 3), (2, 2), (5, 1)])
def test_tensor_contraction_matches_oracle_and_fma(oracle, cfg, F):
    w = configs.CONFIGS[cfg]() if cfg != 4 else configs.config4(frames=F)
    arr, p, rx = w.array, w.params, w.receive
    rf = np.stack([configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=60 + f)
                   for f in range(F)])
    tc_tr = _traces(w, rf, True)
    fma_tr = _traces(w, rf, False)
    assert rel_l2(tc_tr, fma_tr) <= 5e-6
    for f in range(min(F, 2)):
        ref = oracle.decompose_f64(rf[f], arr.sampling_frequency, arr.positions, rx.angles, p.sound_speed)
        assert rel_l2(tc_tr[f], ref) <= 1e-5, (cfg, f)


def test_tensor_contraction_rejects_asymmetric_geometry():
    import ctypes

    arr = kb.TransducerArray(16, 0.3e-3, 5e6, 20e6, 0.6)
    ang = np.array([0.01, 0.05, 0.09])   # no +-theta pairs: the general (non-symmetric) contraction
    h = ctypes.c_void_p()
    _lib.call("kkb_decomposer_create", 2, arr.num_elements, 256, arr.positions.ctypes.data,
              ang.ctypes.data, 3, 20e6, C, 1, ctypes.byref(h))
    try:
        assert _lib.load().kkb_decomposer_symmetric_classes(h) == 0
        with pytest.raises(kb.KKBeamError):
            _lib.call("kkb_decomposer_set_contraction", h, _lib.KKB_CONTRACT_TENSOR)
    finally:
        _lib.load().kkb_decomposer_destroy(h)


def test_tensor_contraction_odd_elements_and_edge_bins(oracle):
    """Odd element count (the middle element has no mirror), a bin count
    that leaves a partial 4-bin tile, and rows beyond a 64-row tile."""
    arr = kb.TransducerArray(37, 0.3e-3, 5e6, 20e6, 0.6)
    T = 250                                  # K = 126 bins: the last tile is half empty
    params = kb.AcquisitionParams(C, np.linspace(-0.15, 0.15, 9), T)
    rx = kb.uniform_vernier_angles(9, 7, 10 * DEG, 1)
    grid = kb.ImageGrid(-1e-3, 2e-3, 0.1e-3, 0.1e-3, 4, 4)
    w = configs.Workload("odd", arr, params, rx, grid)
    rf = np.stack([configs.noise_rf(9, 37, T, seed=70 + f) for f in range(8)])   # 72 rows
    tc_tr = _traces(w, rf, True)
    fma_tr = _traces(w, rf, False)
    assert rel_l2(tc_tr, fma_tr) <= 1e-6
    ref = oracle.decompose_f64(rf[7], arr.sampling_frequency, arr.positions, rx.angles, C)
    assert rel_l2(tc_tr[7], ref) <= 1e-5
