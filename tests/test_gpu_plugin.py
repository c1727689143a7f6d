"""The reference-side binding (kkbeam_plugin): shims with the exact numba
kernel signatures, and install()/restore() on a kkbeam-shaped namespace
(the reference itself is not present on the GPU box)."""

import sys
import types

import numpy as np
import pytest

from conftest import C, golden, rel_l2

pytestmark = pytest.mark.gpu

from paper_2603_22496_b200 import kkbeam_plugin  # noqa: E402


def test_kk_kernel_shim_matches_reference_image():
    g = golden("config1")
    out = np.empty((128, 128), dtype=np.complex128)
    fs, t0 = 20e6, 6e-6
    kkbeam_plugin.kk_kernel(g["compressed"], g["ltx"], g["ltz"], g["lrx"], g["lrz"], np.ones(11),
                            fs, (0.0 - t0) * fs, True, out)
    assert rel_l2(out, g["image"]) <= 1e-5
    kkbeam_plugin.kk_kernel(g["compressed"], g["ltx"], g["ltz"], g["lrx"], g["lrz"], g["weights"],
                            fs, (0.3e-6 - t0) * fs, False, out)
    assert rel_l2(out, g["image_nearest"]) <= 1e-5


def test_das_kernel_shim_matches_reference_image(oracle, point_dataset):
    arr, params, rf, grid = point_dataset
    g = golden("das_point")
    an = oracle.analytic_signal(rf)
    ltx, ltz = oracle.tx_tables(grid.x, grid.z, params.transmit_angles, C)
    out = np.empty((64, 64), dtype=np.complex128)
    kkbeam_plugin.das_kernel(an, ltx, ltz, g["hyp"], g["base"], g["frac"], grid.x, grid.z,
                             arr.positions, np.inf, np.ones(64), arr.sampling_frequency, 0.0,
                             True, out)
    assert rel_l2(out, g["image"]) <= 1e-5


def test_install_rebinds_and_restores():
    pkg = types.ModuleType("kkbeam")
    bf = types.ModuleType("kkbeam.beamform")
    cp = types.ModuleType("kkbeam.compress")
    sentinel = object()
    bf._kk_kernel = bf._das_kernel = cp.shear_and_sum = sentinel
    saved = {k: sys.modules.get(k) for k in ("kkbeam", "kkbeam.beamform", "kkbeam.compress")}
    sys.modules.update({"kkbeam": pkg, "kkbeam.beamform": bf, "kkbeam.compress": cp})
    try:
        h = kkbeam_plugin.install(pkg)
        assert bf._kk_kernel is kkbeam_plugin.kk_kernel
        assert bf._das_kernel is kkbeam_plugin.das_kernel
        assert cp.shear_and_sum is kkbeam_plugin.shear_and_sum
        h.restore()
        assert bf._kk_kernel is sentinel and cp.shear_and_sum is sentinel
    finally:
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v


def test_render_traces_shim_is_bit_identical(oracle):
    # the numba signature of _render_traces (simulate.py:187-220): the shim adds
    # the echoes into the caller's float32 array, like the reference
    from conftest import sha

    import paper_2603_22496_b200 as kb
    from paper_2603_22496_b200 import configs

    w = configs.config1()
    g = golden("config1")
    arr, p = w.array, w.params
    out = np.zeros((p.num_transmits, arr.num_elements, p.num_samples), np.float32)
    kkbeam_plugin.render_traces(out, g["phantom_x"], g["phantom_z"], np.ones(5), arr.positions,
                                np.sin(p.transmit_angles), np.cos(p.transmit_angles),
                                1.0 / p.sound_speed, arr.sampling_frequency, p.start_time,
                                g["pulse"], float((g["pulse"].size - 1) // 2), False)
    out += 1e-3 * np.random.default_rng(0).standard_normal(out.shape, dtype=np.float32)
    assert sha(out) == str(g["rf_sha"])
    assert kb.simulate_rf is not None


def test_gamma_match_shim_matches_reference():
    import os

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_display_golden import images

    import paper_2603_22496_b200 as kb

    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "display.npz"))
    grid, a, b = images(kb, 0)
    g, m = kkbeam_plugin.gamma_match(kb.IntensityImage(a, grid), kb.IntensityImage(b, grid))
    assert abs(g - float(G["gamma_0"])) <= 1e-12
    with pytest.raises(kb.MetricError):
        kkbeam_plugin.gamma_match(kb.IntensityImage(np.zeros_like(a), grid), kb.IntensityImage(b, grid))
