"""Analytic-signal conversion on the GPU (drop-in for kkbeam.spectral).

``analytic_signal`` keeps the reference signature and container contract
(spectral.py:84-93): float32 RF (N, L, T) in, complex64 one-sided data out;
the FFT -> one-sided weights -> inverse FFT runs as libkkb kernels
(real-pair packed Stockham FFT, weights and 1/T folded into the spectral
write, inverse FFT over the non-negative bins only).
"""

from __future__ import annotations

import numpy as np

from . import _device as dev
from . import _lib
from .core import IQ_DTYPE, AnalyticRF, RFVolume
from .errors import ConfigError


def one_sided_weights(num_samples: int) -> np.ndarray:
    """Spectral weights of the analytic signal (spectral.py:65-81):
    1 at DC, 2 on positive bins, 1 at Nyquist for even T, 0 on negative bins."""
    if num_samples < 1:
        raise ConfigError("need at least one sample")
    w = np.zeros(num_samples)
    pos_end = (num_samples + 1) // 2  # first bin that is not strictly positive
    w[1:pos_end] = 2.0
    w[0] = 1.0
    if num_samples % 2 == 0:
        w[num_samples // 2] = 1.0
    return w


def analytic_signal_device(rf, out=None, stream=None):
    """(..., T) float32 CUDA tensor -> complex64 CUDA tensor, asynchronous."""
    t = dev.require_cuda()
    if rf.dtype != t.float32:
        raise ConfigError("analytic_signal_device expects float32 RF")
    rf = rf.contiguous()
    T = int(rf.shape[-1])
    if out is None:
        out = t.empty(rf.shape, dtype=t.complex64, device=rf.device)
    _lib.call("kkb_analytic_signal", dev.ptr(rf), rf.numel() // T, T, dev.ptr(out),
              dev.stream_handle(stream))
    return out


def analytic_signal(rf: RFVolume) -> AnalyticRF:
    """Convert raw RF to its analytic signal, trace by trace, on the GPU."""
    x = dev.to_device(rf.data)
    out = analytic_signal_device(x)
    dev.synchronize()
    return AnalyticRF(dev.to_host(out).astype(IQ_DTYPE, copy=False), rf.array, rf.params)
