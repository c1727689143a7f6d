"""CPU-side checks: the C ABI library loads and exports every declared
symbol; host-side mirror of the reference interface (containers, sampling
objects, validation, error mapping, workload geometry).  No kernel runs."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import C, DEG, ROOT, golden

import paper_2603_22496_b200 as kb
from paper_2603_22496_b200 import _lib, configs
from paper_2603_22496_b200.errors import ConfigError, GeometryError, GuardBandError, DataError


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "kkb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kkb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_hot_path():
    names = _declared_symbols()
    for must in ("kkb_kk", "kkb_das", "kkb_analytic_signal", "kkb_shear_and_sum",
                 "kkb_build_kk_luts", "kkb_decomposer_create", "kkb_decomposer_run",
                 "kkb_kk_plan_run", "kkb_log_compress", "kkb_compound", "kkb_kk_taps"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in _declared_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert _lib.version().startswith("kkb-b200")
    assert isinstance(_lib.launch_count(), int)


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_oracle_library_exports():
    from oracle import kkbeam_oracle as O

    O.build()
    lib = ctypes.CDLL(O._LIB_PATH)
    for name in ("oracle_kk_kernel", "oracle_das_kernel", "oracle_render_traces"):
        assert hasattr(lib, name)


# ------------------------------------------------------------------ sampling
def test_sampling_matches_reference_goldens():
    g = golden("sampling")
    d75 = 32 * DEG / 74
    got = {
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
    for k, v in got.items():
        assert np.array_equal(v, g[k]), k


def test_sampling_validation():
    with pytest.raises(ConfigError):
        kb.transmit_angles(1, 0.1)
    with pytest.raises(ConfigError):
        kb.uniform_vernier_angles(7, 5, 0.2, 4)  # j > floor(N/2)
    with pytest.raises(ConfigError):
        kb.confocal_angles(2, 5, 0.2)
    with pytest.raises(ConfigError):
        kb.explicit_angles([0.1, 0.2])  # not symmetric
    even = kb.uniform_vernier_angles(7, 4, 12 * DEG, 1)
    assert 0.0 not in even.angles and even.num_angles == 4
    assert len(kb.support(kb.transmit_angles(3, 0.1), even, 5e6, C)) == 12


# ------------------------------------------------------------------ containers
def test_container_validation(small_array):
    params = kb.AcquisitionParams(C, [0.0, 0.1], 128)
    with pytest.raises(GeometryError):
        kb.RFVolume(np.zeros((3, 64, 128), np.float32), small_array, params)
    with pytest.raises(GeometryError):
        kb.RFVolume(np.zeros((2, 63, 128), np.float32), small_array, params)
    bad = np.zeros((2, 64, 128), np.float32)
    bad[0, 0, 0] = np.nan
    with pytest.raises(DataError):
        kb.RFVolume(bad, small_array, params)
    rf = kb.RFVolume(np.zeros((2, 64, 128)), small_array, params)
    assert rf.data.dtype == np.float32 and not rf.data.flags.writeable
    rx = kb.explicit_angles([-0.1, 0.0, 0.1])
    with pytest.raises(ConfigError):
        kb.CompressedRF(np.zeros((2, 3, 128), np.complex64), rx, params)
    rfc = kb.CompressedRF(np.zeros((2, 3, 128), np.complex64), rx, params, small_array)
    assert rfc.sampling_frequency == small_array.sampling_frequency
    with pytest.raises(ConfigError):
        kb.AcquisitionParams(C, [0.1, 0.0], 128)
    with pytest.raises(ConfigError):
        kb.ImageGrid(0, 0, 1e-4, 1e-4, 4, 4)
    with pytest.raises(ConfigError):
        kb.TransducerArray(64, 0.3e-3, 5e6, 10e6, 0.6)


def test_beamform_config_and_cache_model():
    with pytest.raises(ConfigError):
        kb.BeamformConfig(interpolation="cubic")
    with pytest.raises(ConfigError):
        kb.BeamformConfig(max_rx_angle=math.pi / 2)
    grid = kb.ImageGrid(-5e-3, 5e-3, 0.057e-3, 0.056e-3, 180, 180)
    assert kb.cache_model_entries(grid, 15, 21, "kk") == 12960
    assert kb.cache_model_entries(grid, 15, 192, "das") == 72360
    with pytest.raises(ConfigError):
        kb.cache_model_entries(grid, 15, 21, "mv")


def test_compression_ratio_and_guard_band():
    assert round(kb.compression_ratio(192, 7), 1) == 27.4
    assert round(kb.compression_ratio(192, 57), 1) == 3.4
    with pytest.raises(ConfigError):
        kb.compression_ratio(0, 7)
    ap = 191 * 0.23e-3
    assert kb.guard_band_samples(ap, 23.8 * DEG, 20.83e6, C) == int(
        np.ceil(ap * np.sin(23.8 * DEG) * 20.83e6 / C))
    assert kb.guard_band_samples(ap, 0.0, 20.83e6, C) == 0


def test_guard_band_error_is_raised_before_any_device_work(small_array):
    # validation happens on the host, so this runs without a GPU
    params = kb.AcquisitionParams(C, [0.0, 0.1], 256)
    an = kb.AnalyticRF(np.zeros((2, 64, 256), np.complex64), small_array, params)
    rx = kb.explicit_angles([-0.4, 0.0, 0.4])
    guard = kb.guard_band_samples(63 * 0.23e-3, 0.4, small_array.sampling_frequency, C)
    with pytest.raises(GuardBandError) as err:
        kb.compress(an, rx, last_used_sample=256 - guard + 5)
    assert "5 more trailing samples" in str(err.value)


def test_status_mapping():
    from paper_2603_22496_b200.errors import DeviceError, raise_for_status

    raise_for_status(0, "x")
    with pytest.raises(ConfigError):
        raise_for_status(-1, "x")
    with pytest.raises(GeometryError):
        raise_for_status(-2, "x")
    with pytest.raises(DeviceError):
        raise_for_status(-3, "x")


def test_one_sided_weights_host():
    assert list(kb.one_sided_weights(8)) == [1, 2, 2, 2, 1, 0, 0, 0]
    assert list(kb.one_sided_weights(7)) == [1, 2, 2, 2, 0, 0, 0]
    with pytest.raises(ConfigError):
        kb.one_sided_weights(0)


# ------------------------------------------------------------------ workloads
def test_workload_sizes_match_survey():
    w1, w2, w4, w5 = configs.config1(), configs.config2(), configs.config4(), configs.config5()
    assert w1.pixel_pairs == 128 * 128 * 121
    assert w2.pairs == 75 and w2.grid.nx * w2.grid.nz == 102_400
    assert w4.pairs == 121 and w4.frames == 400 and w4.params.num_samples == 1536
    assert w5.pairs == 961 and w5.grid.nx * w5.grid.nz == 2_097_152
    w3 = configs.config3()
    assert {k: v[0].num_transmits * v[1].num_angles for k, v in w3.extra_receive.items()} == {
        "dense_vernier": 81, "shifted_vernier": 75, "confocal": 75, "hybrid": 125}


def test_plugin_install_on_the_real_reference():
    """install() rebinds the reference's own kernel globals (no kernel runs)."""
    import sys

    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference package not present (GPU box)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, src)
    try:
        import kkbeam

        from paper_2603_22496_b200 import kkbeam_plugin

        bf, cp = sys.modules["kkbeam.beamform"], sys.modules["kkbeam.compress"]
        sim = sys.modules["kkbeam.simulate"]
        import kkbeam.cli  # noqa: F401  (the CLI imports gamma_match by name)

        met, cli = sys.modules["kkbeam.metrics"], sys.modules["kkbeam.cli"]
        orig = (bf._kk_kernel, bf._das_kernel, cp.shear_and_sum, sim._render_traces)
        orig_g = (met.gamma_match, cli.gamma_match)
        h = kkbeam_plugin.install(kkbeam)
        assert met.gamma_match is kkbeam_plugin.gamma_match
        assert cli.gamma_match is kkbeam_plugin.gamma_match
        assert bf._kk_kernel is kkbeam_plugin.kk_kernel
        assert bf._das_kernel is kkbeam_plugin.das_kernel
        assert cp.shear_and_sum is kkbeam_plugin.shear_and_sum
        assert sim._render_traces is kkbeam_plugin.render_traces
        # the package-level name keeps the float64 original (oracle stays intact)
        assert kkbeam.shear_and_sum is orig[2]
        h.restore()
        assert (bf._kk_kernel, bf._das_kernel, cp.shear_and_sum, sim._render_traces) == orig
        assert (met.gamma_match, cli.gamma_match) == orig_g
    finally:
        sys.path.remove(src)


def test_no_device_means_loud_failure(monkeypatch):
    # the product path refuses to run without CUDA instead of falling back
    from paper_2603_22496_b200 import _device
    from paper_2603_22496_b200.errors import DeviceError

    t = _device.torch()
    if t.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(DeviceError):
        kb.analytic_signal(kb.RFVolume(np.zeros((1, 4, 64)), kb.TransducerArray(
            4, 0.23e-3, 5.2e6, 20.83e6, 0.67), kb.AcquisitionParams(C, [0.0], 64)))


def test_bench_roofline_helpers_read_the_committed_profiles():
    """bench.py's roofline denominators come from committed measurements
    (profiles/): the shared-memory (LDS.128) and FP32 peaks, the L2 read
    bandwidth and the gather's ncu DRAM traffic."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    l2 = bench._l2_roofline(24000.0)
    assert l2["bound"] == "l2" and 16000 < l2["peak"] < 20000 and 1.2 < l2["frac"] < 1.6
    t = bench._gather_traffic(400)
    # between the L2-warm single-block capture (0.55 GB) and the gather's
    # compulsory bytes plus slack (traces 0.60 GB + IQ 0.21 GB + tables + planes)
    assert 0.3e9 < t < 1.2e9
    assert bench._gather_traffic(200) == t / 2
    smem, fp32, kind = bench._onchip_peaks()
    assert kind == "measured" and 30000 < smem < 40000 and 60 < fp32 < 80
    # both arms report the same config object
    from paper_2603_22496_b200 import configs

    w = configs.config4(frames=400)
    c = bench._config(w, 400, 1)
    assert c["workload"] == w.name and c["pixel_pairs_per_frame"] == 256 * 256 * 121


def test_numa_cpulist_parsing_and_pci_address():
    from types import SimpleNamespace

    from paper_2603_22496_b200._numa import parse_cpulist, pci_address

    assert parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert parse_cpulist("5") == [5]
    assert parse_cpulist("") == []
    props = SimpleNamespace(pci_domain_id=0, pci_bus_id=0x1b, pci_device_id=0)
    assert pci_address(props) == "0000:1b:00.0"
