"""KKRF binary RF container (I/O formats and ingest).

Mirrors the reference's ``kkbeam.rffile`` (rffile.py): the same layout,
``write_container`` / ``read_container`` with the same validation order,
error types and messages, so files round-trip bit-exactly between the two
packages.  The bytes move through libkkb's native reader/writer
(``kkb_kkrf_*``, csrc/kkrf.cu); ``read_container_device`` /
``read_ensemble_device`` stream payloads straight into HBM (disk reads
overlapped with host->device copies) for the throughput path.

Layout (little-endian; rffile.py:1-26):
    0  4  magic b"KKRF"      4  2  u16 version (1)     6  1  u8 kind
    7  4  u32 N             11  4  u32 channels        15  4  u32 T
   19  8  f64 fs            27  8  f64 fc              35  8  f64 c
   43  8  f64 pitch         51  8  f64 t0
   59  8N f64 transmit angles, then 8M f64 receive angles (kind 2 only),
   then the payload (N, channels, T): float32 (kind 0) or complex64 (1, 2).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import AcquisitionParams, AnalyticRF, CompressedRF, RFVolume, TransducerArray
from .errors import ConfigError, FileFormatError
from .sampling import ReceiveAngleSet, explicit_angles

MAGIC = b"KKRF"
VERSION = 1
KIND_REAL = 0
KIND_ANALYTIC = 1
KIND_COMPRESSED = 2
HEAD_BYTES = 59


def _placeholder_bandwidth(fs: float, fc: float) -> float:
    """Widest fractional bandwidth the sampling rate supports, capped at 1
    (the header does not record it; rffile.py:52-58)."""
    bw = (fs / fc - 2.0) / 2.0
    if bw <= 0:
        raise FileFormatError(f"sampling frequency {fs} cannot support center frequency {fc}")
    return min(1.0, bw)


def _kind_of(container) -> int:
    for cls, kind in ((RFVolume, KIND_REAL), (AnalyticRF, KIND_ANALYTIC),
                      (CompressedRF, KIND_COMPRESSED)):
        if isinstance(container, cls):
            return kind
    raise FileFormatError(f"cannot serialize {type(container).__name__}")


def _header(kind, shape, fs, fc, c, pitch, t0) -> _lib.KKRFHeader:
    h = _lib.KKRFHeader()
    h.magic = MAGIC
    h.version = VERSION
    h.kind = kind
    h.num_transmits, h.num_channels, h.num_samples = (int(v) for v in shape)
    h.sampling_frequency, h.center_frequency = float(fs), float(fc)
    h.sound_speed, h.pitch, h.start_time = float(c), float(pitch), float(t0)
    h.head_bytes = HEAD_BYTES
    return h


def _geometry_of(container, kind):
    """(fs, fc, pitch) as write_container records them (rffile.py:77-92)."""
    if kind == KIND_COMPRESSED:
        arr = container.array
        return (container.sampling_frequency, arr.center_frequency if arr is not None else 0.0,
                arr.pitch if arr is not None else 0.0)
    arr = container.array
    return arr.sampling_frequency, arr.center_frequency, arr.pitch


def write_container(path, container) -> None:
    """Serialize an RF container to `path` (layout above)."""
    kind = _kind_of(container)
    data = np.ascontiguousarray(container.data)
    fs, fc, pitch = _geometry_of(container, kind)
    p = container.params
    h = _header(kind, data.shape, fs, fc, p.sound_speed, pitch, p.start_time)
    tx = np.ascontiguousarray(p.transmit_angles, dtype="<f8")
    rx = (np.ascontiguousarray(container.receive_angles.angles, dtype="<f8")
          if kind == KIND_COMPRESSED else None)
    _lib.call("kkb_kkrf_write", os.fsencode(path), ctypes.byref(h), tx.ctypes.data,
              None if rx is None else rx.ctypes.data, data.ctypes.data, data.nbytes, 0, None)


@dataclass(frozen=True)
class _Parsed:
    kind: int
    shape: tuple
    fs: float
    fc: float
    c: float
    pitch: float
    t0: float
    tx: np.ndarray
    rx: np.ndarray | None
    payload_offset: int
    dtype: np.dtype


def _read_host(path, offset, nbytes) -> bytes:
    buf = ctypes.create_string_buffer(max(int(nbytes), 1))
    if nbytes:
        _lib.call("kkb_kkrf_read_bytes", os.fsencode(path), int(offset), int(nbytes),
                  ctypes.addressof(buf), 0, None)
    return buf.raw[:nbytes]


def _parse(path) -> _Parsed:
    """Head + angle tables with read_container's checks, in its order
    (rffile.py:122-151)."""
    h = _lib.KKRFHeader()
    lib = _lib.load()
    st = lib.kkb_kkrf_read_header(os.fsencode(path), ctypes.byref(h))
    if st == -6:
        raise FileFormatError(f"{path}: truncated header")
    if st:
        _lib.raise_for_status(st, "kkb_kkrf_read_header", _lib.last_error())
    magic = bytes(h.magic)
    n, channels, t = h.num_transmits, h.num_channels, h.num_samples
    fs, fc, c, pitch, t0 = (h.sampling_frequency, h.center_frequency, h.sound_speed, h.pitch,
                            h.start_time)
    if magic != MAGIC:
        raise FileFormatError(f"{path}: bad magic {magic!r}")
    if h.version != VERSION:
        raise FileFormatError(f"{path}: unsupported format version {h.version}")
    if h.kind not in (KIND_REAL, KIND_ANALYTIC, KIND_COMPRESSED):
        raise FileFormatError(f"{path}: unknown kind byte {h.kind}")
    if min(n, channels, t) <= 0:
        raise FileFormatError(f"{path}: bad dimensions {(n, channels, t)}")
    if fs <= 0 or c <= 0:
        raise FileFormatError(f"{path}: nonpositive sampling frequency or sound speed")
    if h.kind != KIND_COMPRESSED and (pitch <= 0 or fc <= 0):
        raise FileFormatError(f"{path}: nonpositive pitch or center frequency")
    size = h.file_bytes
    pos = HEAD_BYTES
    tables = 8 * n + (8 * channels if h.kind == KIND_COMPRESSED else 0)
    blob = _read_host(path, pos, min(tables, max(size - pos, 0)))
    # the reference reads tx with np.frombuffer (a short file raises its ValueError)
    tx = np.frombuffer(blob, dtype="<f8", count=n, offset=0).copy()
    pos += 8 * n
    rx = None
    if h.kind == KIND_COMPRESSED:
        if size < pos + 8 * channels:
            raise FileFormatError(f"{path}: truncated receive angle table")
        rx = np.frombuffer(blob, dtype="<f8", count=channels, offset=8 * n).copy()
        pos += 8 * channels
    dtype = np.dtype("<f4") if h.kind == KIND_REAL else np.dtype("<c8")
    expected = pos + n * channels * t * dtype.itemsize
    if size != expected:
        raise FileFormatError(f"{path}: payload size mismatch (have {size}, expected {expected})")
    return _Parsed(int(h.kind), (n, channels, t), fs, fc, c, pitch, t0, tx, rx, pos, dtype)


def _metadata(path, ps: _Parsed):
    """(params, array, receive) exactly as read_container builds them."""
    n, channels, t = ps.shape
    params = AcquisitionParams(sound_speed=ps.c, transmit_angles=ps.tx, num_samples=t,
                               start_time=ps.t0)
    if ps.kind == KIND_COMPRESSED:
        dthi = float(ps.tx[1] - ps.tx[0]) if n > 1 else 0.0
        try:
            receive = explicit_angles(ps.rx, dthi)
        except ConfigError as exc:
            raise FileFormatError(f"{path}: bad receive angle table ({exc})") from exc
        return params, None, receive
    array = TransducerArray(num_elements=channels, pitch=ps.pitch, center_frequency=ps.fc,
                            sampling_frequency=ps.fs,
                            fractional_bandwidth=_placeholder_bandwidth(ps.fs, ps.fc))
    return params, array, None


def read_container(path):
    """Load a container written by write_container: RFVolume, AnalyticRF or
    CompressedRF by the kind byte; FileFormatError for anything malformed."""
    ps = _parse(path)
    nbytes = int(np.prod(ps.shape)) * ps.dtype.itemsize
    data = np.empty(ps.shape, dtype=ps.dtype)
    _lib.call("kkb_kkrf_read_bytes", os.fsencode(path), ps.payload_offset, nbytes,
              data.ctypes.data, 0, None)
    params, array, receive = _metadata(path, ps)
    if ps.kind == KIND_COMPRESSED:
        return CompressedRF(data=data, receive_angles=receive, params=params, array=None,
                            sampling_frequency=ps.fs)
    cls = RFVolume if ps.kind == KIND_REAL else AnalyticRF
    return cls(data=data, array=array, params=params)


@dataclass(frozen=True, eq=False)
class DeviceContainer:
    """A KKRF container whose payload lives in HBM (CUDA tensor)."""

    kind: int
    data: object
    params: AcquisitionParams
    array: TransducerArray | None
    receive_angles: ReceiveAngleSet | None
    sampling_frequency: float


def _payload_tensor(shape, dtype):
    from . import _device as dev

    return dev.empty(shape, np.float32 if dtype == np.dtype("<f4") else np.complex64)


def read_container_device(path, stream=None) -> DeviceContainer:
    """read_container with the payload streamed into device memory."""
    from . import _device as dev

    ps = _parse(path)
    params, array, receive = _metadata(path, ps)
    out = _payload_tensor(ps.shape, ps.dtype)
    _lib.call("kkb_kkrf_read_bytes", os.fsencode(path), ps.payload_offset,
              out.numel() * out.element_size(), dev.ptr(out), 1, dev.stream_handle(stream))
    return DeviceContainer(ps.kind, out, params, array, receive, ps.fs)


def read_ensemble_device(paths, stream=None, threads: int | None = None):
    """Frames stored one per KKRF file (same kind and geometry) -> one
    (F, N, channels, T) device tensor, e.g. the input of KKEngine.run.
    ``threads`` parallel readers (default: up to 8, one per file at most)
    stream the files through pinned staging into HBM
    (``kkb_kkrf_read_ensemble``).  Returns (tensor, metadata of the first file)."""
    from . import _device as dev

    paths = list(paths)
    if not paths:
        raise ConfigError("read_ensemble_device needs at least one file")
    parsed = [_parse(p) for p in paths]
    first = parsed[0]
    for p, ps in zip(paths[1:], parsed[1:]):
        if (ps.kind, ps.shape, ps.fs, ps.c, ps.t0) != (first.kind, first.shape, first.fs, first.c,
                                                       first.t0) or not np.array_equal(ps.tx, first.tx):
            raise FileFormatError(f"{p}: geometry differs from {paths[0]}")
    params, array, receive = _metadata(paths[0], first)
    out = _payload_tensor((len(paths),) + first.shape, first.dtype)
    frame_bytes = int(np.prod(first.shape)) * first.dtype.itemsize
    names = [ctypes.c_char_p(os.fsencode(p)) for p in paths]
    arr_p = (ctypes.c_char_p * len(names))(*names)
    offs = (ctypes.c_longlong * len(parsed))(*[ps.payload_offset for ps in parsed])
    n_threads = int(threads) if threads else min(8, len(paths), os.cpu_count() or 1)
    _lib.call("kkb_kkrf_read_ensemble", ctypes.cast(arr_p, ctypes.c_void_p),
              ctypes.cast(offs, ctypes.c_void_p), len(paths), frame_bytes, dev.ptr(out),
              max(1, n_threads), dev.stream_handle(stream))
    return out, DeviceContainer(first.kind, None, params, array, receive, first.fs)


def write_container_device(path, like, data, stream=None) -> None:
    """Write a device payload `data` (CUDA tensor shaped like like.data) with
    the metadata of container `like` (e.g. frames of an ensemble)."""
    from . import _device as dev

    kind = like.kind if isinstance(like, DeviceContainer) else _kind_of(like)
    want = np.float32 if kind == KIND_REAL else np.complex64
    if tuple(data.shape) != tuple(like.data.shape if like.data is not None else data.shape) \
            or data.dtype != dev._dtype(want):
        raise FileFormatError("payload shape/dtype does not match the container")
    if isinstance(like, DeviceContainer):
        fs = like.sampling_frequency
        fc = like.array.center_frequency if like.array is not None else 0.0
        pitch = like.array.pitch if like.array is not None else 0.0
        rx_set = like.receive_angles
    else:
        fs, fc, pitch = _geometry_of(like, kind)
        rx_set = like.receive_angles if kind == KIND_COMPRESSED else None
    p = like.params
    h = _header(kind, data.shape, fs, fc, p.sound_speed, pitch, p.start_time)
    tx = np.ascontiguousarray(p.transmit_angles, dtype="<f8")
    rx = np.ascontiguousarray(rx_set.angles, dtype="<f8") if kind == KIND_COMPRESSED else None
    _lib.call("kkb_kkrf_write", os.fsencode(path), ctypes.byref(h), tx.ctypes.data,
              None if rx is None else rx.ctypes.data, dev.ptr(data),
              data.numel() * data.element_size(), 1, dev.stream_handle(stream))
