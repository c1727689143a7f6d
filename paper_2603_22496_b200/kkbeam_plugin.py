"""Reference-side binding: route the reference package's own kernels to libkkb.

The reference (`kkbeam`) has no FFI; its wrappers look up these module
globals at call time:

* ``kkbeam.beamform._kk_kernel``   (beamform.py:212-236, called at 363-374)
* ``kkbeam.beamform._das_kernel``  (beamform.py:178-209, called at 281-297)
* ``kkbeam.compress.shear_and_sum`` (compress.py:54-82, called at 120)
* ``analytic_signal`` (spectral.py:84-93; bound by name in ``kkbeam``,
  ``kkbeam.spectral`` and ``kkbeam.cli``)
* ``kkbeam.simulate._render_traces`` (simulate.py:187-220, called at 280-293;
  the forward simulator, §8(f) row 4 — bit-identical on the GPU)
* ``kkbeam.metrics.gamma_match`` and the CLI's imported name
  ``kkbeam.cli.gamma_match`` (metrics.py:175-202, called at cli.py:167; the
  display map, §8(f) row 2)
* ``kkbeam.bench._kk_stage_fns`` / ``_das_stage_fns`` (bench.py:113-153,
  91-110; used by ``bench_kk`` / ``bench_das`` and ``kkbeam bench``): the
  staged benchmark's stages on the device (``paper_2603_22496_b200.bench``)

The shims below have exactly those signatures (flat numpy arrays in, the
caller's ``out`` array filled in place) and run the sm_100a kernels through
the C ABI.  ``install(kkbeam)`` rebinds the globals, so ``kkbeam.kk``,
``kkbeam.das`` and ``kkbeam.compress`` — and the reference's own test suite,
via ``-p paper_2603_22496_b200.pytest_kkbeam_gpu`` — run on the GPU with no
change to the reference source.  See INTEGRATION.md.
"""

from __future__ import annotations

import sys

import numpy as np

from . import _device as dev
from . import _lib


def _launch_kk(data, ltx, ltz, lrx, lrz, weights, fs, shift, linear, out):
    # plan cached across calls on the same tables (beamform._KKPlanCache):
    # one H2D of the traces, one gather launch, one D2H of the image per call
    from .beamform import kk_plans

    kk_plans.run_host(data, (ltx, ltz, lrx, lrz), weights, fs, shift, linear, out)


def kk_kernel(data, ltx, ltz, lrx, lrz, weights, fs, shift, linear, out):
    """Drop-in for kkbeam.beamform._kk_kernel (same arguments, fills `out`)."""
    _launch_kk(np.asarray(data, dtype=np.complex64), ltx, ltz, lrx, lrz, weights, fs, shift,
               linear, out)


def das_kernel(data, ltx, ltz, hyp, base, frac, xcoord, zcoord, upos, tan_max, weights, fs,
               shift, linear, out):
    """Drop-in for kkbeam.beamform._das_kernel (same arguments, fills `out`)."""
    t = dev.require_cuda()
    arrs = [dev.to_device(np.ascontiguousarray(a)) for a in
            (np.asarray(data, dtype=np.complex64), ltx, ltz, hyp)]
    bd = dev.to_device(np.ascontiguousarray(base, dtype=np.int64))
    rest = [dev.to_device(np.ascontiguousarray(a, dtype=np.float64)) for a in
            (frac, xcoord, zcoord, upos, weights)]
    n, l, T = data.shape
    nx, nz = out.shape
    o = t.empty((nx, nz), dtype=t.complex128, device="cuda")
    _lib.call("kkb_das", dev.ptr(arrs[0]), n, l, T, dev.ptr(arrs[1]), dev.ptr(arrs[2]),
              dev.ptr(arrs[3]), int(hyp.shape[0]), dev.ptr(bd), dev.ptr(rest[0]), dev.ptr(rest[1]),
              dev.ptr(rest[2]), dev.ptr(rest[3]), float(tan_max), dev.ptr(rest[4]), float(fs),
              float(shift), int(bool(linear)), nx, nz, dev.ptr(o), _lib.KKB_OUT_C128,
              dev.stream_handle())
    dev.synchronize()
    out[...] = dev.to_host(o)


def analytic_signal(rf):
    """Drop-in for kkbeam.spectral.analytic_signal (spectral.py:84-93): the
    one-sided FFT -> weights -> inverse FFT on the GPU (K1 + K3), returned
    in the reference's own AnalyticRF container (so its validation and
    isinstance checks are unchanged)."""
    from .spectral import analytic_signal_device

    core = sys.modules.get("kkbeam.core")
    x = dev.to_device(np.ascontiguousarray(rf.data, dtype=np.float32))
    out = dev.to_host(analytic_signal_device(x))
    if core is None:  # not installed against the reference: this package's container
        from .core import AnalyticRF
    else:
        AnalyticRF = core.AnalyticRF
    return AnalyticRF(out, rf.array, rf.params)


def shear_and_sum(data, sampling_frequency, positions, angles, sound_speed):
    """Drop-in for kkbeam.compress.shear_and_sum (complex128 (N, M, T) out)."""
    from .compress import shear_and_sum as gpu_shear

    return gpu_shear(data, sampling_frequency, positions, angles, sound_speed)


def render_traces(out, sx, sz, refl, upos, sin_t, cos_t, inv_c, fs, t0, wave, half, spread):
    """Drop-in for kkbeam.simulate._render_traces: adds the echoes to `out`
    (float32 (N, L, T), in place), bit-identical to the numba kernel."""
    n_tx, n_el, n_t = out.shape
    d_out = dev.to_device(np.ascontiguousarray(out, dtype=np.float32))
    arrs = [dev.to_device(np.ascontiguousarray(a, dtype=np.float64)) for a in
            (sx, sz, refl, upos, sin_t, cos_t, wave)]
    _lib.call("kkb_render_traces", dev.ptr(d_out), n_tx, n_el, n_t, dev.ptr(arrs[0]),
              dev.ptr(arrs[1]), dev.ptr(arrs[2]), int(np.asarray(sx).size), dev.ptr(arrs[3]),
              dev.ptr(arrs[4]), dev.ptr(arrs[5]), float(inv_c), float(fs), float(t0),
              dev.ptr(arrs[6]), int(np.asarray(wave).size), float(half), int(bool(spread)),
              dev.stream_handle())
    dev.synchronize()
    out[...] = dev.to_host(d_out)


def gamma_match(image, reference, lo=0.1, hi=1.0, tol=1e-3):
    """Drop-in for kkbeam.metrics.gamma_match: the golden-section search with
    every objective evaluated on the device; raises the reference's own
    MetricError for all-zero images."""
    if image.pixels.max() <= 0 or reference.pixels.max() <= 0:
        err = sys.modules.get("kkbeam.errors")
        exc = getattr(err, "MetricError", None) if err is not None else None
        if exc is None:
            from .errors import MetricError as exc
        raise exc("gamma matching needs nonzero images")
    from .display import gamma_match as device_gamma_match

    return device_gamma_match(image, reference, lo, hi, tol)


class Installed:
    """Handle returned by install(); ``restore()`` puts the originals back."""

    def __init__(self, saved):
        self._saved = saved

    def restore(self):
        for (mod, name), value in self._saved.items():
            setattr(mod, name, value)
        self._saved = {}


def install(kkbeam_pkg=None, spectral: bool = True) -> Installed:
    """Rebind the reference's kernel globals to the GPU shims (and, with
    `spectral`, its analytic_signal: the whole README pipeline
    analytic_signal -> compress -> kk then runs on the GPU).

    Note kkbeam/__init__.py:34 binds ``kkbeam.compress`` to the *function*,
    so the submodule is taken from sys.modules."""
    if kkbeam_pkg is None:
        import kkbeam as kkbeam_pkg  # noqa: F401  (the reference package)
    bf = sys.modules["kkbeam.beamform"]
    cp = sys.modules["kkbeam.compress"]
    saved = {(bf, "_kk_kernel"): bf._kk_kernel, (bf, "_das_kernel"): bf._das_kernel,
             (cp, "shear_and_sum"): cp.shear_and_sum}
    bf._kk_kernel = kk_kernel
    bf._das_kernel = das_kernel
    cp.shear_and_sum = shear_and_sum
    if spectral:  # analytic_signal is imported by name into kkbeam and kkbeam.cli too
        for name in ("kkbeam.spectral", "kkbeam", "kkbeam.cli"):
            mod = sys.modules.get(name)
            if mod is not None and hasattr(mod, "analytic_signal"):
                saved[(mod, "analytic_signal")] = mod.analytic_signal
                mod.analytic_signal = analytic_signal
    sim = sys.modules.get("kkbeam.simulate")
    if sim is not None and hasattr(sim, "_render_traces"):
        saved[(sim, "_render_traces")] = sim._render_traces
        sim._render_traces = render_traces
    for name in ("kkbeam.metrics", "kkbeam.cli"):
        mod = sys.modules.get(name)
        if mod is not None and hasattr(mod, "gamma_match"):
            saved[(mod, "gamma_match")] = mod.gamma_match
            mod.gamma_match = gamma_match
    # the staged benchmark (bench.py:91-185, `kkbeam bench`): its private
    # stage builders call scipy / numpy directly, so they are rebound to the
    # device stages (paper_2603_22496_b200.bench)
    bm = sys.modules.get("kkbeam.bench")
    if bm is not None and hasattr(bm, "_kk_stage_fns"):
        from . import bench as gpu_bench

        saved[(bm, "_kk_stage_fns")] = bm._kk_stage_fns
        saved[(bm, "_das_stage_fns")] = bm._das_stage_fns
        bm._kk_stage_fns = gpu_bench.kk_stage_fns
        bm._das_stage_fns = gpu_bench.das_stage_fns
    return Installed(saved)
