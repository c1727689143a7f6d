"""The five synthetic workloads of BASELINE.json, in reference terms.

The paper's Verasonics / CIRS-040GSE datasets are not available, so seeded
synthetic inputs with the configs' shapes stand in for them (SURVEY.md
§8(d)).  Each builder returns the geometry only (array, acquisition,
receive set(s), grid); RF comes from ``noise_rf`` (the reference's
``bench.noise_volume``, bench.py:188-194) for throughput, or from the
oracle simulator in the tests for point-target parity.

Resolutions of BASELINE.json ambiguities (also recorded in DESIGN.md):

* config 1: ``start_time = 6 us`` (at t0 = 0 the reference simulator raises
  WindowOverflowError for the seeded scatterers), pulse bw 0.44.
* config 2: KK transmits are every 5th of the 75 DAS transmits starting at
  index 2 (15 angles at 5 Delta); receive angles explicit Delta*[-2..2].
* config 3: the four schemes re-expressed with the reference's own sampling
  objects (dense / shifted vernier, Eq. 9 confocal, hybrid union).
* config 4: ``transmit_angles(11, 10 deg)``; grid z from 5 mm at lambda/4 so
  the image fits the T=1536 window; 400 frames per rank.
* config 5: ``transmit_angles(31, 15 deg)`` x ``confocal_angles(31, 31, 15 deg)``.

Media (``config2_medium``, ``config4_vessel_frame``): the BASELINE phantoms
re-expressed with the reference's own phantom objects (simulate.py:136-184)
and rendered by the GPU forward simulator (bit-identical to the reference's
``_render_traces``): speckle at 10 scatterers per resolution cell with real
N(0, 1) amplitudes (``Phantom.reflectivity`` is real, so BASELINE's "complex
Gaussian amplitudes" are not representable), two anechoic 2 mm cysts, a row
of six amplitude-20 wires, int16 quantisation (``quantize_int16``); the
config-4 ensemble adds a 2 mm vessel whose scatterers move 50 um per frame
(RF linearity: static background + per-frame vessel echoes).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import AcquisitionParams, ImageGrid, TransducerArray
from .sampling import (ReceiveAngleSet, confocal_angles, explicit_angles, transmit_angles,
                       uniform_vernier_angles)

C = 1540.0
DEG = np.pi / 180.0


@dataclass(frozen=True, eq=False)
class Workload:
    name: str
    array: TransducerArray
    params: AcquisitionParams
    receive: ReceiveAngleSet
    grid: ImageGrid
    frames: int = 1
    extra_receive: dict = field(default_factory=dict)  # label -> (params, receive)

    @property
    def pairs(self) -> int:
        return self.params.num_transmits * self.receive.num_angles

    @property
    def pixel_pairs(self) -> int:
        return self.grid.nx * self.grid.nz * self.pairs


def config1() -> Workload:
    arr = TransducerArray(64, 0.3e-3, 5e6, 20e6, 0.44)
    tmax = 10 * DEG
    params = AcquisitionParams(C, transmit_angles(11, tmax), 1024, start_time=6e-6)
    rx = uniform_vernier_angles(11, 11, tmax, 0)
    grid = ImageGrid(-9.6e-3, 5e-3, 19.2e-3 / 127, 40e-3 / 127, 128, 128)
    return Workload("config1_point_targets", arr, params, rx, grid)


def config1_phantom(seed: int = 0):
    """5 unit point scatterers, x in [-8, 8] mm, z in [10, 40] mm."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-8e-3, 8e-3, 5)
    z = rng.uniform(10e-3, 40e-3, 5)
    return x, z, np.ones(5)


def _tx75():
    return transmit_angles(75, 16 * DEG)


def config2() -> Workload:
    arr = TransducerArray(128, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    tx75 = _tx75()
    d = tx75[1] - tx75[0]
    params = AcquisitionParams(C, tx75[2::5], 2048)
    rx = explicit_angles(d * np.array([-2.0, -1.0, 0.0, 1.0, 2.0]), d)
    a = arr.aperture
    lam = C / arr.center_frequency
    grid = ImageGrid(-a / 2, 5e-3, a / 255, lam / 4, 256, 400)
    das_params = AcquisitionParams(C, tx75, 2048)
    return Workload("config2_phantom_vernier", arr, params, rx, grid,
                    extra_receive={"das75": (das_params, None)})


def config3() -> Workload:
    base = config2()
    arr = base.array
    tx75 = _tx75()
    d = tx75[1] - tx75[0]
    lam = C / arr.center_frequency
    a = arr.aperture
    grid = ImageGrid(-a / 2, 5e-3, a / 383, lam / 5, 384, 512)
    dense_p = AcquisitionParams(C, tx75[1::9], 2048)
    dense_rx = uniform_vernier_angles(9, 9, 36 * d, 0)
    shift_p = AcquisitionParams(C, tx75[2::5], 2048)
    shifted_rx = uniform_vernier_angles(15, 5, 35 * d, 7)
    confocal_rx = confocal_angles(15, 5, 35 * d)
    hyb_p = AcquisitionParams(C, tx75[1::3], 2048)
    hyb_rx = explicit_angles(np.concatenate([confocal_angles(25, 3, 36 * d).angles,
                                             uniform_vernier_angles(25, 2, 36 * d, 0).angles]),
                             3 * d)
    extra = {
        "dense_vernier": (dense_p, dense_rx),
        "shifted_vernier": (shift_p, shifted_rx),
        "confocal": (shift_p, confocal_rx),
        "hybrid": (hyb_p, hyb_rx),
    }
    return Workload("config3_scheme_sweep", arr, hyb_p, hyb_rx, grid, extra_receive=extra)


def config4(frames: int = 400) -> Workload:
    arr = TransducerArray(128, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    tmax = 10 * DEG
    params = AcquisitionParams(C, transmit_angles(11, tmax), 1536)
    rx = uniform_vernier_angles(11, 11, tmax, 0)
    a = arr.aperture
    lam = C / arr.center_frequency
    grid = ImageGrid(-a / 2, 5e-3, a / 255, lam / 4, 256, 256)
    return Workload("config4_fus_ensemble", arr, params, rx, grid, frames=frames)


def config5() -> Workload:
    arr = TransducerArray(256, 0.2e-3, 7.5e6, 30e6, 0.6)
    tmax = 15 * DEG
    params = AcquisitionParams(C, transmit_angles(31, tmax), 4096)
    rx = confocal_angles(31, 31, tmax)
    a = arr.aperture
    lam = C / arr.center_frequency
    grid = ImageGrid(-a / 2, 2e-3, a / 1023, 0.12 * lam, 1024, 2048)
    return Workload("config5_large_aperture", arr, params, rx, grid)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def noise_rf(n_tx: int, n_el: int, n_t: int, seed: int = 0) -> np.ndarray:
    """Seeded float32 white-noise RF (the reference's bench.noise_volume)."""
    return np.random.default_rng(seed).standard_normal((n_tx, n_el, n_t), dtype=np.float32)


# ------------------------------------------------------------------ media
def speckle_density(array: TransducerArray, z_mid: float) -> float:
    """10 scatterers per resolution cell: cell = (lambda z /
    aperture) x (pulse length / 2), pulse length c / (bw fc); per m^2."""
    lam = C / array.center_frequency
    lateral = lam * z_mid / array.aperture
    axial = C / (array.fractional_bandwidth * array.center_frequency) / 2.0
    return 10.0 / (lateral * axial)


CYSTS_C2 = ((-8e-3, 14e-3), (7e-3, 24e-3))      # (x, z) of the two 2 mm anechoic cysts
WIRES_C2_DEPTH = 19e-3                           # six wires, 5 mm apart, amplitude 20


def config2_medium(seed: int = 0, z_range=(5e-3, 33e-3)):
    """Config-2 calibration-phantom medium: speckle over
    the aperture width x z_range, two 2 mm anechoic cysts, six wires."""
    from .simulate import Phantom, merge_phantoms, speckle_phantom, wire_phantom

    arr = config2().array
    a = arr.aperture
    z0, z1 = z_range
    sp = speckle_phantom((-a / 2, a / 2, z0, z1), speckle_density(arr, 0.5 * (z0 + z1)), seed,
                         inclusion_center=CYSTS_C2[0], inclusion_radius=2e-3)
    cx, cz = CYSTS_C2[1]
    keep = (sp.x - cx) ** 2 + (sp.z - cz) ** 2 > (2e-3) ** 2
    sp = Phantom(sp.x[keep], sp.z[keep], sp.reflectivity[keep])
    wires = wire_phantom([5e-3] * 5, WIRES_C2_DEPTH, 20.0)
    return merge_phantoms(sp, wires)


def quantize_int16(rf: np.ndarray):
    """BASELINE config 2's sample format: q = clip(round(rf / s), +-32767)
    with s = max|rf| / 32767 (the oracle consumes q.astype(float32))."""
    s = float(np.abs(rf).max()) / 32767.0
    return np.clip(np.round(rf / s), -32767, 32767).astype(np.int16), s


VESSEL_Z = 15e-3          # centre depth of the config-4 vessel (2 mm diameter, lateral)
VESSEL_STEP = 50e-6       # lateral displacement of its scatterers per frame


def config4_background(seed: int = 0):
    """Static config-4 medium: the config-2 speckle cropped to z <= 24 mm
    (T = 1536 window), the vessel lumen carved out."""
    from .simulate import Phantom, speckle_phantom

    arr = config4().array
    a = arr.aperture
    sp = speckle_phantom((-a / 2, a / 2, 5e-3, 24e-3), speckle_density(arr, 14.5e-3), seed)
    keep = np.abs(sp.z - VESSEL_Z) > 1e-3
    return Phantom(sp.x[keep], sp.z[keep], sp.reflectivity[keep])


def config4_vessel_frame(frame: int, seed: int = 1, amplitude: float = 0.5):
    """Moving scatterers of the 2 mm vessel in frame `frame`: seeded positions
    inside the lumen over the central half of the aperture, shifted laterally
    by 50 um per frame (wrapped within that span)."""
    from .simulate import Phantom

    arr = config4().array
    h = arr.aperture / 4
    rng = np.random.default_rng(seed)
    count = int(round(speckle_density(arr, VESSEL_Z) * 2 * h * 2e-3))
    x = rng.uniform(-h, h, count)
    z = rng.uniform(VESSEL_Z - 1e-3, VESSEL_Z + 1e-3, count)
    r = amplitude * rng.standard_normal(count)
    x = (x + h + VESSEL_STEP * frame) % (2 * h) - h
    return Phantom(x, z, r)
