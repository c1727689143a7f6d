"""Display mapping, image writers and the guard-band budget.

* ``gamma_match`` mirrors metrics.py:175-202: the exponent search runs the
  reference's golden-section steps (metrics.py:156-172) with every objective
  evaluation a device reduction (``kkb_gamma_match``), so a display map of a
  whole ensemble never leaves HBM (``gamma_match_device``).
* ``write_pgm16`` / ``write_raw_f32`` are the reference's output formats
  (cli.py:134-147), byte for byte; ``write_display`` is its per-image flow
  (cli.py:150-174: raw intensity + gamma-matched 16-bit PGM).
* ``last_read_sample`` is cli.py:110-128 — the last sample the kk gather can
  read on a grid, which the reference passes to ``compress`` as
  ``last_used_sample`` — evaluated on the device, bit-identical.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _device as dev
from . import _lib
from .core import AcquisitionParams, ImageGrid, IntensityImage
from .errors import MetricError


def _max_dev(t) -> float:
    out = ctypes.c_double()
    _lib.call("kkb_max_f64", dev.ptr(t), t.numel(), ctypes.byref(out), dev.stream_handle())
    return out.value


def gamma_match_device(image, reference, lo: float = 0.1, hi: float = 1.0, tol: float = 1e-3):
    """(gamma, (image/max)^gamma) for float64 CUDA tensors of one shape."""
    if image.numel() != reference.numel() or image.numel() == 0:
        raise MetricError("gamma matching needs two nonempty images of one size")
    if _max_dev(image) <= 0 or _max_dev(reference) <= 0:
        raise MetricError("gamma matching needs nonzero images")
    g = ctypes.c_double()
    mapped = dev.empty(tuple(image.shape), np.float64)
    _lib.call("kkb_gamma_match", dev.ptr(image), dev.ptr(reference), image.numel(), float(lo),
              float(hi), float(tol), ctypes.byref(g), dev.ptr(mapped), dev.stream_handle())
    return float(g.value), mapped


def gamma_match(image: IntensityImage, reference: IntensityImage, lo: float = 0.1,
                hi: float = 1.0, tol: float = 1e-3) -> tuple[float, np.ndarray]:
    """Exponent matching an image's display brightness to a reference
    (metrics.py:175-202); returns (gamma, mapped image in [0, 1])."""
    im = dev.to_device(image.pixels, np.float64)
    ref = dev.to_device(reference.pixels, np.float64)
    g, mapped = gamma_match_device(im, ref, lo, hi, tol)
    return g, dev.to_host(mapped)


def write_pgm16(path: str, mapped: np.ndarray) -> None:
    """16-bit big-endian binary PGM, rows = depth, columns = lateral (cli.py:134-141)."""
    m = np.clip(np.asarray(mapped, dtype=np.float64), 0.0, 1.0)
    raster = np.round(m.T * 65535.0).astype(">u2")
    nz, nx = raster.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{nx} {nz}\n65535\n".encode("ascii"))
        f.write(raster.tobytes())


def write_raw_f32(path: str, pixels: np.ndarray) -> None:
    """Raw little-endian float32, C order (nx, nz) (cli.py:144-147)."""
    with open(path, "wb") as f:
        f.write(np.ascontiguousarray(pixels, dtype="<f4").tobytes())


def write_display(stem: str, image: IntensityImage, reference: IntensityImage | None = None):
    """cli.py:150-174 for one image: `stem`.f32 raw intensity and `stem`.pgm
    gamma-matched to `reference` (itself when absent or all zero).  Returns
    (gamma, [paths])."""
    ref = reference if reference is not None else image
    if image.pixels.max() <= 0:
        gamma, mapped = 1.0, np.zeros_like(image.pixels)
    else:
        if ref.pixels.max() <= 0:
            ref = image
        gamma, mapped = gamma_match(image, ref)
    write_raw_f32(stem + ".f32", image.pixels)
    write_pgm16(stem + ".pgm", mapped)
    return gamma, [stem + ".f32", stem + ".pgm"]


def last_read_sample(grid: ImageGrid, params: AcquisitionParams, receive_sets, fs: float,
                     pulse_delay: float = 0.0) -> int:
    """Largest sample index the kk beamformer reads on `grid` for the union of
    `receive_sets` (ReceiveAngleSet or (label, set) pairs) -- cli.py:110-128."""
    rx = []
    for item in receive_sets:
        rs = item[1] if isinstance(item, tuple) else item
        rx.extend(float(a) for a in rs.angles)
    tx = [float(a) for a in params.transmit_angles]
    # the reference takes math.sin / math.cos of each angle (not np.sin)
    arrs = [np.array([math.sin(a) for a in tx]), np.array([math.cos(a) for a in tx]),
            np.array([math.sin(a) for a in rx]), np.array([math.cos(a) for a in rx])]
    d = [dev.to_device(a, np.float64) for a in [grid.x, grid.z] + arrs]
    out = ctypes.c_double()
    _lib.call("kkb_last_read_sample_max", dev.ptr(d[0]), grid.nx, dev.ptr(d[1]), grid.nz,
              dev.ptr(d[2]), dev.ptr(d[3]), len(tx), dev.ptr(d[4]), dev.ptr(d[5]), len(rx),
              ctypes.byref(out), dev.stream_handle())
    tau_max = out.value / params.sound_speed
    return int(math.ceil((tau_max + pulse_delay - params.start_time) * fs)) + 1
