"""Receive decomposition on the GPU (drop-in for kkbeam.compress).

Same signatures, guard-band rule and error text as the reference
(compress.py:40-121).  The shear-and-sum runs as libkkb kernels: forward
FFT of every element trace, per-bin contraction over elements with the
phase ramps exp(2 pi i f u_l sin(theta_m) / c) (built in float64, stored
complex64), inverse FFT.  Arithmetic is float32 with float64-accurate
twiddles and ramps (the storage precision of the reference's compress
output, compress.py:121); ``shear_and_sum`` returns that result upcast to
complex128 to keep the reference's return type.
"""

from __future__ import annotations

import math

import numpy as np

from . import _device as dev
from . import _lib
from .core import IQ_DTYPE, AnalyticRF, CompressedRF
from .errors import ConfigError, GuardBandError
from .sampling import ReceiveAngleSet


def compression_ratio(num_elements: int, num_receive: int) -> float:
    """L / M (compress.py:40-44)."""
    if num_elements < 1 or num_receive < 1:
        raise ConfigError("element and receive counts must be positive")
    return num_elements / num_receive


def guard_band_samples(aperture: float, max_abs_angle: float, sampling_frequency: float,
                       sound_speed: float) -> int:
    """Trailing zero samples that absorb the largest shear (compress.py:47-51)."""
    return int(math.ceil(aperture * math.sin(abs(max_abs_angle)) * sampling_frequency / sound_speed))


class _ShearPlanCache:
    """Shear plans (the phase ramps of one geometry, built once in float64)
    keyed by the bytes of (positions, angles, fs, c, T): a reference loop that
    compresses frame after frame pays the ramp build once."""

    def __init__(self, capacity: int = 4):
        from collections import OrderedDict

        self._d = OrderedDict()
        self.capacity = capacity

    def get(self, pos: np.ndarray, ang: np.ndarray, fs: float, c: float, T: int):
        import ctypes

        key = (pos.tobytes(), ang.tobytes(), float(fs), float(c), int(T))
        h = self._d.get(key)
        if h is not None:
            self._d.move_to_end(key)
            return h
        h = ctypes.c_void_p()
        _lib.call("kkb_shear_plan_create", pos.ctypes.data, ang.ctypes.data, int(pos.size), int(ang.size),
                  int(T), float(fs), float(c), ctypes.byref(h))
        self._d[key] = h
        while len(self._d) > self.capacity:
            _, old = self._d.popitem(last=False)
            dev.synchronize()
            _lib.load().kkb_shear_plan_destroy(old)
        return h


shear_plans = _ShearPlanCache()


def shear_and_sum_device(data, sampling_frequency, positions, angles, sound_speed, out=None,
                         stream=None):
    """complex64 CUDA tensor (N, L, T) -> complex64 CUDA tensor (N, M, T)."""
    t = dev.require_cuda()
    if data.dim() != 3:
        raise ConfigError("expected (transmits, elements, samples) data")
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    ang = np.ascontiguousarray(angles, dtype=np.float64)
    if data.shape[1] != pos.size:
        raise ConfigError("element count does not match positions")
    if data.dtype != t.complex64:
        data = data.to(t.complex64)
    data = data.contiguous()
    n, l, T = (int(s) for s in data.shape)
    if out is None:
        out = t.empty((n, ang.size, T), dtype=t.complex64, device=data.device)
    plan = shear_plans.get(pos, ang, sampling_frequency, sound_speed, T)
    _lib.call("kkb_shear_plan_run", plan, dev.ptr(data), n, dev.ptr(out), dev.stream_handle(stream))
    return out


def shear_and_sum(data, sampling_frequency: float, positions, angles, sound_speed: float) -> np.ndarray:
    """(N, L, T) -> (N, M, T) complex128: element l advanced by u_l sin(theta)/c
    in the frequency domain, then summed over elements (compress.py:54-82)."""
    arr = np.asarray(data)
    if arr.ndim != 3:
        raise ConfigError("expected (transmits, elements, samples) data")
    if arr.shape[1] != np.asarray(positions).size:
        raise ConfigError("element count does not match positions")
    x = dev.to_device(arr.astype(np.complex64, copy=False))
    out = shear_and_sum_device(x, sampling_frequency, positions, angles, sound_speed)
    dev.synchronize()
    return dev.to_host(out).astype(np.complex128)


def compress(rf: AnalyticRF, receive: ReceiveAngleSet, last_used_sample: int | None = None) -> CompressedRF:
    """Decompose analytic element data into M virtual plane-wave traces."""
    fs = rf.array.sampling_frequency
    c = rf.params.sound_speed
    if last_used_sample is not None:
        guard = guard_band_samples(rf.array.aperture, float(np.max(np.abs(receive.angles))), fs, c)
        total = rf.params.num_samples
        if total < last_used_sample + guard:
            raise GuardBandError(
                f"window of {total} samples leaves no shear guard band: reading up to "
                f"sample {last_used_sample} needs {last_used_sample + guard - total} "
                "more trailing samples")
    x = dev.to_device(rf.data)
    out = shear_and_sum_device(x, fs, rf.array.positions, receive.angles, c)
    dev.synchronize()
    return CompressedRF(dev.to_host(out).astype(IQ_DTYPE, copy=False), receive, rf.params, rf.array)
