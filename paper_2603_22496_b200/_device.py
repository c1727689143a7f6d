"""Device plumbing: torch CUDA tensors as allocations, streams as handles.

PyTorch provides the caching allocator, streams and pinned host memory;
every computation on those buffers is a libkkb kernel.
"""

from __future__ import annotations

import numpy as np

from .errors import DeviceError

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t

        _torch = _t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise DeviceError("no CUDA device: this package runs its hot path only on the GPU "
                          "(no CPU fallback)")
    return t


_NP2T = None


def _dtype(np_dtype):
    t = torch()
    table = {
        np.dtype(np.float32): t.float32,
        np.dtype(np.float64): t.float64,
        np.dtype(np.complex64): t.complex64,
        np.dtype(np.complex128): t.complex128,
        np.dtype(np.int64): t.int64,
        np.dtype(np.int16): t.int16,
        np.dtype(np.int32): t.int32,
        np.dtype(np.uint32): t.int32,
    }
    return table[np.dtype(np_dtype)]


def to_device(a: np.ndarray, dtype=None):
    """Contiguous host array -> CUDA tensor (synchronous copy)."""
    t = require_cuda()
    a = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    return t.from_numpy(a.copy() if not a.flags.writeable else a).to("cuda")


def empty(shape, np_dtype):
    t = require_cuda()
    return t.empty(tuple(int(s) for s in shape), dtype=_dtype(np_dtype), device="cuda")


def zeros(shape, np_dtype):
    t = require_cuda()
    return t.zeros(tuple(int(s) for s in shape), dtype=_dtype(np_dtype), device="cuda")


def ptr(x) -> int:
    """Device address of a CUDA tensor (None -> NULL)."""
    if x is None:
        return None
    if not x.is_cuda:
        raise DeviceError("expected a CUDA tensor")
    if not x.is_contiguous():
        raise DeviceError("expected a contiguous tensor")
    return x.data_ptr()


def stream_handle(stream=None) -> int:
    """cudaStream_t of `stream` (default: torch's current stream)."""
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return s.cuda_stream


def to_host(x) -> np.ndarray:
    return x.cpu().numpy()


def synchronize(stream=None):
    t = torch()
    if stream is None:
        t.cuda.current_stream().synchronize()
    else:
        stream.synchronize()
