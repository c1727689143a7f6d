"""Display / budgeting goldens produced by the REFERENCE itself.

Run in the build container (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_display_golden.py

Stores: the bytes of cli.write_pgm16 / cli.write_raw_f32 for a fixed array,
metrics.gamma_match on two seeded intensity images, and cli._last_read_sample
(called with a minimal config object exposing the four accessors it uses)
for two geometries.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def images(kb, seed):
    rng = np.random.default_rng(seed)
    grid = kb.ImageGrid(-5e-3, 4e-3, 0.2e-3, 0.1e-3, 64, 48)
    a = rng.gamma(0.7, size=(64, 48)) ** 2
    b = rng.gamma(1.3, size=(64, 48))
    return grid, a, b


class _Cfg:
    """The accessors cli._last_read_sample reads (cli.py:110-128)."""

    def __init__(self, kb, grid, params, array, pulse_delay):
        self._g, self._p, self._a = grid, params, array
        self._b = kb.BeamformConfig(pulse_delay=pulse_delay)

    def grid(self):
        return self._g

    def acquisition(self):
        return self._p

    def array(self):
        return self._a

    def beamform_config(self):
        return self._b


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF_SRC)
    import kkbeam as kb
    from kkbeam import cli, metrics

    out = {}
    mapped = np.linspace(-0.2, 1.3, 35).reshape(7, 5)
    with tempfile.TemporaryDirectory() as d:
        cli.write_pgm16(os.path.join(d, "m.pgm"), mapped)
        cli.write_raw_f32(os.path.join(d, "m.f32"), mapped)
        out["pgm_bytes"] = np.frombuffer(open(os.path.join(d, "m.pgm"), "rb").read(), np.uint8)
        out["f32_bytes"] = np.frombuffer(open(os.path.join(d, "m.f32"), "rb").read(), np.uint8)
    out["mapped_in"] = mapped
    for seed in (0, 1):
        grid, a, b = images(kb, seed)
        g, m = metrics.gamma_match(kb.IntensityImage(a, grid), kb.IntensityImage(b, grid))
        out[f"gamma_{seed}"] = np.float64(g)
        out[f"gamma_mapped_{seed}"] = m
    cases = [
        (kb.TransducerArray(64, 0.3e-3, 5e6, 20e6, 0.44),
         kb.AcquisitionParams(1540.0, kb.transmit_angles(11, np.deg2rad(10)), 1024, start_time=6e-6),
         [kb.uniform_vernier_angles(11, 11, np.deg2rad(10), 0)],
         kb.ImageGrid(-9.6e-3, 5e-3, 19.2e-3 / 127, 40e-3 / 127, 128, 128), 0.0),
        (kb.TransducerArray(128, 0.3e-3, 5.2e6, 20.8e6, 0.6),
         kb.AcquisitionParams(1540.0, kb.transmit_angles(15, np.deg2rad(14)), 2048),
         [kb.confocal_angles(15, 5, np.deg2rad(14)),
          kb.uniform_vernier_angles(15, 5, np.deg2rad(14), 7)],
         kb.ImageGrid(-19e-3, 5e-3, 38.1e-3 / 255, 0.074e-3, 256, 400), 0.7e-6),
    ]
    for i, (arr, params, sets, grid, pd) in enumerate(cases):
        out[f"last_read_{i}"] = np.int64(cli._last_read_sample(
            _Cfg(kb, grid, params, arr, pd), [(f"s{j}", s) for j, s in enumerate(sets)]))
    np.savez_compressed(os.path.join(OUT, "display.npz"), **out)
    print({k: (v if v.size == 1 else v.shape) for k, v in out.items()})


if __name__ == "__main__":
    main()
