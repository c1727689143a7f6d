"""The reference's staged throughput benchmark (kkbeam/bench.py), on the GPU.

The reference splits both pipelines into four timed stages —
``reorg_fft`` (FFT of the RF along time), ``hilbert_compress`` (one-sided
weights; for KK also the per-angle phase-and-sum over elements), ``ifft``
and ``beamform`` — and reports the median wall time per stage over
``repetitions`` runs after a discarded first one (bench.py:1-19, 63-75).

``kk_stage_fns`` / ``das_stage_fns`` below have the signatures of the
reference's ``_kk_stage_fns`` / ``_das_stage_fns`` (bench.py:113-153,
91-110) and return the same (stage name, fn(state)) list, each stage one
step of the device path:

    reorg_fft          pinned H2D of the RF + K1 (real FFT)
    hilbert_compress   KK: K2, the contraction with the one-sided weights
                       folded into the cached ramps; DAS: the weights
    ifft               K3 (inverse FFT)
    beamform           K5 (KK gather) / K7 (DAS) + D2H of the image

Every stage ends with a device synchronisation, so the host wall clock the
reference takes around it covers the stage's GPU work.  As in the reference,
delay tables and ramps are built once outside the timed stages (plans are
created when the stage list is built); the RF is staged into pinned host
memory there too, the way an acquisition buffer would arrive.

``kkbeam_plugin.install`` rebinds the reference's two private builders to
these, so the reference's own ``bench_kk`` / ``bench_das`` and its ``kkbeam
bench`` command time the GPU path unmodified.  ``bench_kk`` / ``bench_das``
here return a ``StageTimings`` with the reference's fields for this
package's containers.
"""

from __future__ import annotations

import ctypes
import sys
import time
from dataclasses import dataclass

import numpy as np

from . import _device as dev
from . import _lib
from .errors import ConfigError

STAGES = ("reorg_fft", "hilbert_compress", "ifft", "beamform")


@dataclass(frozen=True)
class StageTimings:
    """Median per-stage wall time (ms) of one benchmark row; the fields of
    kkbeam.bench.StageTimings (bench.py:46-69)."""

    label: str
    method: str
    num_channels: int
    compression_ratio: float
    lut_entries: int
    reorg_fft_ms: float
    hilbert_compress_ms: float
    ifft_ms: float
    beamform_ms: float

    def stage_ms(self, name: str) -> float:
        return float(getattr(self, name + "_ms"))

    @property
    def total_ms(self) -> float:
        return float(sum(self.stage_ms(s) for s in STAGES))


def _image_class(luts):
    """ComplexImage of the package the LUT set comes from (the reference's
    when called through the plugin, this package's otherwise)."""
    mod = sys.modules.get(type(luts).__module__)
    cls = getattr(mod, "ComplexImage", None) if mod is not None else None
    if cls is None:
        from .core import ComplexImage as cls
    return cls


def _weights(bconf, count):
    w = getattr(bconf, "channel_weights", None)
    if w is None:
        return None
    w = np.asarray(w, dtype=np.float64)
    if w.shape != (count,):
        raise ConfigError(f"channel_weights must have shape ({count},)")
    return w


def _pinned_rf(rf):
    t = dev.require_cuda()
    host = t.from_numpy(np.array(rf.data, dtype=np.float32, copy=True)).pin_memory()  # containers are read-only
    return host, t.empty(host.shape, dtype=t.float32, device="cuda")


def kk_stage_fns(rf, receive, luts, bconf):
    """GPU form of kkbeam.bench._kk_stage_fns (bench.py:113-153)."""
    from .beamform import kk_plans

    t = dev.require_cuda()
    N, L, T = rf.data.shape
    M = receive.num_angles
    fs = rf.array.sampling_frequency
    c = rf.params.sound_speed
    rf_h, rf_d = _pinned_rf(rf)
    traces = t.empty((N, M, T), dtype=t.complex64, device="cuda")
    pos = np.ascontiguousarray(rf.array.positions, dtype=np.float64)
    ang = np.ascontiguousarray(receive.angles, dtype=np.float64)
    dec = ctypes.c_void_p()
    _lib.call("kkb_decomposer_create", N, L, T, pos.ctypes.data, ang.ctypes.data, M, float(fs), float(c), 1,
              ctypes.byref(dec))
    tables = (luts.lut_tx_x, luts.lut_tx_z, luts.lut_rx_x, luts.lut_rx_z)
    nx, nz = luts.grid.nx, luts.grid.nz
    shift = (bconf.pulse_delay - rf.params.start_time) * fs
    entry = kk_plans.entry(tables, N, M, T, nx, nz, _weights(bconf, M), fs, shift,
                           bconf.interpolation == "linear")
    image_cls = _image_class(luts)
    s = dev.stream_handle()

    def stage(k, state):
        _lib.call("kkb_decomposer_run_stage", dec, k, dev.ptr(rf_d), 1, dev.ptr(traces), s)
        dev.synchronize()

    def reorg_fft(state):
        rf_d.copy_(rf_h, non_blocking=True)
        stage(0, state)

    def hilbert_compress(state):
        stage(1, state)

    def ifft(state):
        stage(2, state)
        state["traces"] = traces

    def beamform(state):
        _lib.call("kkb_kk_plan_run", entry["plan"], dev.ptr(traces), 1, 0, dev.ptr(entry["out_d"]),
                  _lib.KKB_OUT_C128, nx * nz, None, None, s)
        entry["out_h"].copy_(entry["out_d"], non_blocking=True)
        dev.synchronize()
        state["image"] = image_cls(entry["out_h"].numpy().copy(), luts.grid)

    fns = [reorg_fft, hilbert_compress, ifft, beamform]
    # the decomposer plan lives as long as the stage list
    fns[0].plan = _Owner(dec, (rf_h, rf_d, traces, entry))
    return list(zip(STAGES, fns))


def das_stage_fns(rf, luts, bconf):
    """GPU form of kkbeam.bench._das_stage_fns (bench.py:91-110)."""
    import math

    t = dev.require_cuda()
    N, L, T = rf.data.shape
    K = T // 2 + 1
    fs = rf.array.sampling_frequency
    rf_h, rf_d = _pinned_rf(rf)
    spec = t.empty((N * L, K), dtype=t.complex64, device="cuda")
    iq = t.empty((N, L, T), dtype=t.complex64, device="cuda")
    g = luts.grid
    up = {k: dev.to_device(np.ascontiguousarray(getattr(luts, k), dtype=np.float64))
          for k in ("lut_tx_x", "lut_tx_z", "lut_rx_hypot", "rx_frac", "element_positions")}
    base = dev.to_device(np.ascontiguousarray(luts.rx_base, dtype=np.int64))
    xz = (dev.to_device(np.ascontiguousarray(g.x, dtype=np.float64)),
          dev.to_device(np.ascontiguousarray(g.z, dtype=np.float64)))
    w = _weights(bconf, L)
    wd = dev.to_device(w) if w is not None else None
    gate = getattr(bconf, "max_rx_angle", None)
    tan_max = math.tan(gate) if gate is not None else math.inf
    shift = (bconf.pulse_delay - rf.params.start_time) * fs
    out_d = t.empty((g.nx, g.nz), dtype=t.complex128, device="cuda")
    out_h = t.empty((g.nx, g.nz), dtype=t.complex128).pin_memory()
    image_cls = _image_class(luts)
    s = dev.stream_handle()

    def stage(k):
        _lib.call("kkb_analytic_signal_stage", k, dev.ptr(rf_d), N * L, T, dev.ptr(spec), dev.ptr(iq), s)
        dev.synchronize()

    def reorg_fft(state):
        rf_d.copy_(rf_h, non_blocking=True)
        stage(0)

    def hilbert_compress(state):
        stage(1)

    def ifft(state):
        stage(2)
        state["iq"] = iq

    def beamform(state):
        _lib.call("kkb_das", dev.ptr(iq), N, L, T, dev.ptr(up["lut_tx_x"]), dev.ptr(up["lut_tx_z"]),
                  dev.ptr(up["lut_rx_hypot"]), int(luts.lut_rx_hypot.shape[0]), dev.ptr(base),
                  dev.ptr(up["rx_frac"]), dev.ptr(xz[0]), dev.ptr(xz[1]), dev.ptr(up["element_positions"]),
                  float(tan_max), dev.ptr(wd), float(fs), float(shift), int(bconf.interpolation == "linear"),
                  g.nx, g.nz, dev.ptr(out_d), _lib.KKB_OUT_C128, s)
        out_h.copy_(out_d, non_blocking=True)
        dev.synchronize()
        state["image"] = image_cls(out_h.numpy().copy(), g)

    return list(zip(STAGES, (reorg_fft, hilbert_compress, ifft, beamform)))


class _Owner:
    """Destroys the stage list's decomposer plan with it."""

    def __init__(self, handle, keep):
        self.handle, self.keep = handle, keep

    def __del__(self):
        try:
            if self.handle:
                dev.synchronize()
                _lib.load().kkb_decomposer_destroy(self.handle)
        except Exception:  # interpreter shutdown
            pass
        self.handle = None


def time_stages(stage_fns, repetitions: int) -> dict:
    """Median ms per stage over `repetitions` runs after one discarded warm-up
    run (the reference's rule, bench.py:63-75)."""
    if repetitions < 3:
        raise ConfigError("benchmark needs at least 3 repetitions")
    samples = {name: [] for name, _ in stage_fns}
    for rep in range(repetitions + 1):
        state = {}
        for name, fn in stage_fns:
            t0 = time.perf_counter()
            fn(state)
            if rep:
                samples[name].append(time.perf_counter() - t0)
    return {name: 1e3 * float(np.median(v)) for name, v in samples.items()}


def bench_kk(rf, grid, receive, repetitions: int = 3, bconf=None) -> StageTimings:
    """Staged KK benchmark of one receive set on the GPU (bench.py:172-185)."""
    from .beamform import BeamformConfig, build_kk_luts, cache_model_entries
    from .compress import compression_ratio

    bconf = BeamformConfig() if bconf is None else bconf
    luts = build_kk_luts(grid, rf.params, receive)
    ms = time_stages(kk_stage_fns(rf, receive, luts, bconf), repetitions)
    M = receive.num_angles
    return StageTimings(f"kk_m{M}", "kk", M, compression_ratio(rf.array.num_elements, M),
                        cache_model_entries(grid, rf.params.num_transmits, M, "kk"),
                        *(ms[s] for s in STAGES))


def bench_das(rf, grid, repetitions: int = 3, bconf=None) -> StageTimings:
    """Staged DAS benchmark on the GPU (bench.py:156-169)."""
    from .beamform import BeamformConfig, build_das_luts, cache_model_entries

    bconf = BeamformConfig() if bconf is None else bconf
    luts = build_das_luts(grid, rf.array, rf.params)
    ms = time_stages(das_stage_fns(rf, luts, bconf), repetitions)
    L = rf.array.num_elements
    return StageTimings("das", "das", L, 1.0, cache_model_entries(grid, rf.params.num_transmits, L, "das"),
                        *(ms[s] for s in STAGES))


def noise_volume(array, params, seed: int = 0):
    """Seeded white-noise RF volume (N, L, T) float32, the reference's
    throughput input (bench.py:188-194: numpy's default_rng standard normal,
    so the same seed gives the same volume)."""
    from .core import RFVolume

    shape = (params.num_transmits, array.num_elements, params.num_samples)
    data = np.random.default_rng(seed).standard_normal(shape, dtype=np.float32)
    return RFVolume(data=data, array=array, params=params)


def _row_cells(row):
    return [row.label, row.method, row.num_channels, repr(row.compression_ratio), row.lut_entries,
            *(repr(row.stage_ms(s)) for s in STAGES), repr(row.total_ms)]


def write_bench_csv(rows, stream) -> None:
    """Rows as CSV (the reference's columns, bench.py:197-222)."""
    import csv

    w = csv.writer(stream)
    w.writerow(["label", "method", "channels", "compression_ratio", "lut_entries",
                *(s + "_ms" for s in STAGES), "total_ms"])
    for row in rows:
        w.writerow(_row_cells(row))


def bench_csv_text(rows) -> str:
    import io

    buf = io.StringIO()
    write_bench_csv(rows, buf)
    return buf.getvalue()


def format_bench_table(rows) -> str:
    """Fixed-width console table in milliseconds (the reference's layout,
    bench.py:231-245)."""
    head = (f"{'label':<10} {'chan':>5} {'ratio':>7} {'lut':>10} "
            + " ".join(f"{s + '_ms':>19}" for s in STAGES) + f" {'total_ms':>12}")
    out = [head, "-" * len(head)]
    for r in rows:
        out.append(f"{r.label:<10} {r.num_channels:>5} {r.compression_ratio:>7.2f} {r.lut_entries:>10} "
                   + " ".join(f"{r.stage_ms(s):>19.3f}" for s in STAGES) + f" {r.total_ms:>12.3f}")
    return "\n".join(out)
