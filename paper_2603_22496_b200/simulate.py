"""Forward RF simulator on the GPU (harness input).

Mirrors the reference's ``kkbeam.simulate`` interface (simulate.py): point
phantoms, Gaussian pulses and ``simulate_rf``.  The echo rendering — the
reference's numba ``_render_traces`` (simulate.py:187-220), minutes of CPU
time for the config-4/5 speckle media — runs as the K8 CUDA kernel
``kkb_render_traces`` and is bit-identical to it.  Host-side parts stay as
the reference defines them: argument validation, the window-overflow check
(simulate.py:246-264), the pulse (scipy ``gausspulse``, simulate.py:106-133)
and the additive noise (numpy PCG64, simulate.py:293-295), so a simulated
volume equals the reference's sample for sample.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _device as dev
from . import _lib
from .core import RF_DTYPE, AcquisitionParams, RFVolume, TransducerArray
from .errors import ConfigError, GeometryError, WindowOverflowError


class Scatterer(NamedTuple):
    x: float
    z: float
    reflectivity: float = 1.0


def _frozen_f64(a) -> np.ndarray:
    out = np.atleast_1d(np.asarray(a, dtype=np.float64))
    if out.base is not None or not out.flags.owndata:
        out = out.copy()
    out.setflags(write=False)
    return out


@dataclass(frozen=True, eq=False)
class Phantom:
    """Point scatterers as parallel float64 arrays (simulate.py:33-76)."""

    x: np.ndarray
    z: np.ndarray
    reflectivity: np.ndarray

    def __post_init__(self):
        x, z, r = _frozen_f64(self.x), _frozen_f64(self.z), _frozen_f64(self.reflectivity)
        if x.ndim != 1 or x.shape != z.shape or x.shape != r.shape:
            raise ConfigError("phantom arrays must be 1-D and equally sized")
        if x.size and z.min() <= 0:
            raise ConfigError("scatterers must lie below the array (z > 0)")
        object.__setattr__(self, "x", x)
        object.__setattr__(self, "z", z)
        object.__setattr__(self, "reflectivity", r)

    def __len__(self) -> int:
        return int(self.x.size)

    @property
    def scatterers(self) -> list[Scatterer]:
        return [Scatterer(float(a), float(b), float(c))
                for a, b, c in zip(self.x, self.z, self.reflectivity)]

    @classmethod
    def from_scatterers(cls, scatterers) -> "Phantom":
        pts = [Scatterer(*s) for s in scatterers]
        return cls([p.x for p in pts], [p.z for p in pts], [p.reflectivity for p in pts])


def merge_phantoms(a: Phantom, b: Phantom) -> Phantom:
    """a's scatterers first, then b's (simulate.py:79-85)."""
    return Phantom(np.concatenate([a.x, b.x]), np.concatenate([a.z, b.z]),
                   np.concatenate([a.reflectivity, b.reflectivity]))


@dataclass(frozen=True, eq=False)
class Pulse:
    """Time-centred odd-length waveform; peak at index (len-1)/2 (simulate.py:88-102)."""

    center_frequency: float
    fractional_bandwidth: float
    sampling_frequency: float
    waveform: np.ndarray

    def __post_init__(self):
        w = _frozen_f64(self.waveform)
        if w.ndim != 1 or w.size < 3 or w.size % 2 == 0:
            raise ConfigError("pulse waveform must be 1-D with odd length >= 3")
        object.__setattr__(self, "waveform", w)

    @property
    def peak_index(self) -> int:
        return (self.waveform.size - 1) // 2


def make_pulse(center_frequency: float, fractional_bandwidth: float, sampling_frequency: float,
               cutoff_db: float = -60.0) -> Pulse:
    """Gaussian pulse with -6 dB full width fractional_bandwidth * fc,
    truncated at cutoff_db (simulate.py:106-133)."""
    from scipy.signal import gausspulse

    fc, bw, fs = center_frequency, fractional_bandwidth, sampling_frequency
    if fc <= 0 or fs <= 0:
        raise ConfigError("frequencies must be positive")
    if not 0 < bw <= 1:
        raise ConfigError("fractional bandwidth must be in (0, 1]")
    if fs <= 2.0 * fc * (1.0 + bw / 2.0):
        raise ConfigError("sampling frequency does not cover the pulse band")
    if cutoff_db >= 0:
        raise ConfigError("cutoff_db must be negative")
    t_cut = gausspulse("cutoff", fc=fc, bw=bw, bwr=-6, tpr=cutoff_db)
    half = max(1, int(math.ceil(t_cut * fs)))
    t = np.arange(-half, half + 1) / fs
    return Pulse(fc, bw, fs, gausspulse(t, fc=fc, bw=bw, bwr=-6))


def wire_phantom(spacings, depth: float, reflectivity: float = 1.0) -> Phantom:
    """Lateral row of wires at `depth`, centred on x = 0 (simulate.py:136-151)."""
    gaps = np.asarray(spacings, dtype=np.float64)
    if gaps.ndim != 1:
        raise ConfigError("spacings must be a 1-D sequence")
    if gaps.size and gaps.min() <= 0:
        raise ConfigError("wire spacings must be positive")
    if depth <= 0:
        raise ConfigError("depth must be positive")
    x = np.concatenate([[0.0], np.cumsum(gaps)])
    x = x - x[-1] / 2.0
    return Phantom(x, np.full(x.size, depth), np.full(x.size, reflectivity))


def speckle_phantom(region, density: float, seed: int, inclusion_center=None,
                    inclusion_radius: float = 0.0) -> Phantom:
    """Uniform scatterers with N(0, 1) reflectivity in a box, optional anechoic
    disc removed (simulate.py:154-184); same generator draws as the reference."""
    x0, x1, z0, z1 = (float(v) for v in region)
    if not (x1 > x0 and z1 > z0 and z0 > 0):
        raise ConfigError("speckle region must be a nonempty box below the array")
    if density <= 0:
        raise ConfigError("density must be positive")
    count = int(round(density * (x1 - x0) * (z1 - z0)))
    if count < 1:
        raise ConfigError("density too low: no scatterers in region")
    rng = np.random.default_rng(seed)
    x = rng.uniform(x0, x1, count)
    z = rng.uniform(z0, z1, count)
    refl = rng.standard_normal(count)
    if inclusion_center is not None and inclusion_radius > 0:
        cx, cz = (float(v) for v in inclusion_center)
        keep = (x - cx) ** 2 + (z - cz) ** 2 > inclusion_radius ** 2
        x, z, refl = x[keep], z[keep], refl[keep]
    return Phantom(x, z, refl)


def _check_window(array: TransducerArray, params: AcquisitionParams, phantom: Phantom,
                  pulse: Pulse, sin_t, cos_t) -> None:
    """WindowOverflowError for the scatterer needing the most samples
    (latest transmit arrival + farther aperture edge, simulate.py:246-264)."""
    upos = array.positions
    fs = array.sampling_frequency
    tau_in = (phantom.x[:, None] * sin_t[None, :] + phantom.z[:, None] * cos_t[None, :]) \
        / params.sound_speed
    edge = np.maximum(np.hypot(phantom.x - upos[0], phantom.z),
                      np.hypot(phantom.x - upos[-1], phantom.z))
    need = (tau_in.max(axis=1) + edge / params.sound_speed - params.start_time) * fs \
        + pulse.waveform.size
    worst = int(np.argmax(need))
    if need[worst] >= params.num_samples:
        raise WindowOverflowError(
            f"scatterer {worst} at ({phantom.x[worst]:.6g}, {phantom.z[worst]:.6g}) m "
            f"needs {int(math.ceil(need[worst])) + 1} samples, window has {params.num_samples}")


def render_rf_device(array: TransducerArray, params: AcquisitionParams, phantom: Phantom,
                     pulse: Pulse, geometric_spreading: bool = False, out=None, stream=None):
    """Noise-free echo volume (N, L, T) float32 as a CUDA tensor, rendered by
    K8 (bit-identical to the reference's _render_traces).  `out` (optional,
    CUDA float32) is accumulated onto; otherwise a zero volume is used."""
    if pulse.sampling_frequency != array.sampling_frequency:
        raise GeometryError("pulse and array sampling frequencies differ")
    n_tx, n_el, n_t = params.num_transmits, array.num_elements, params.num_samples
    sin_t = np.sin(params.transmit_angles)
    cos_t = np.cos(params.transmit_angles)
    if len(phantom):
        _check_window(array, params, phantom, pulse, sin_t, cos_t)
    if out is None:
        out = dev.zeros((n_tx, n_el, n_t), np.float32)
    if len(phantom):
        d = [dev.to_device(a, np.float64) for a in
             (phantom.x, phantom.z, phantom.reflectivity, array.positions, sin_t, cos_t,
              pulse.waveform)]
        _lib.call("kkb_render_traces", dev.ptr(out), n_tx, n_el, n_t, dev.ptr(d[0]),
                  dev.ptr(d[1]), dev.ptr(d[2]), len(phantom), dev.ptr(d[3]), dev.ptr(d[4]),
                  dev.ptr(d[5]), 1.0 / params.sound_speed, float(array.sampling_frequency),
                  float(params.start_time), dev.ptr(d[6]), int(pulse.waveform.size),
                  float(pulse.peak_index), int(bool(geometric_spreading)),
                  dev.stream_handle(stream))
        dev.synchronize(stream)  # the staging tensors in `d` die with this frame
    return out


def simulate_rf(array: TransducerArray, params: AcquisitionParams, phantom: Phantom, pulse: Pulse,
                noise_rms: float = 0.0, seed: int | None = None,
                geometric_spreading: bool = False) -> RFVolume:
    """Render the RF volume (N transmits, L elements, T samples), as
    simulate.py:223-296: echoes on the GPU, then white noise drawn by numpy
    exactly as the reference draws it."""
    data = dev.to_host(render_rf_device(array, params, phantom, pulse, geometric_spreading))
    if noise_rms > 0.0:
        rng = np.random.default_rng(seed)
        data += noise_rms * rng.standard_normal(data.shape, dtype=RF_DTYPE)
    return RFVolume(data, array, params)
