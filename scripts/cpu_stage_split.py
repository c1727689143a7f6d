"""Per-stage CPU times of one config-4 frame: the reference's own bench stages
(baseline/_ref) next to the oracle port's (diagnostic for the reference arm)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(1, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
import numpy as np  # noqa: E402

import kkbeam as R  # noqa: E402
from kkbeam import bench as RB  # noqa: E402

from oracle import kkbeam_oracle as O  # noqa: E402
from paper_2603_22496_b200 import configs  # noqa: E402

w = configs.config4(frames=1)
g, a, p, rx = w.grid, w.array, w.params, w.receive
arr = R.TransducerArray(a.num_elements, a.pitch, a.center_frequency, a.sampling_frequency,
                        a.fractional_bandwidth)
params = R.AcquisitionParams(p.sound_speed, np.asarray(p.transmit_angles), p.num_samples,
                             start_time=p.start_time)
recv = R.uniform_vernier_angles(11, 11, 10 * np.pi / 180, 0)
grid = R.ImageGrid(g.x0, g.z0, g.dx, g.dz, g.nx, g.nz)
rfa = configs.noise_rf(p.num_transmits, a.num_elements, p.num_samples, seed=0)
rf = R.RFVolume(rfa, arr, params)
luts = R.build_kk_luts(grid, params, recv)
stages = RB._kk_stage_fns(rf, recv, luts, R.BeamformConfig())
REPS = 10
acc = {n: 0.0 for n, _ in stages}
for it in range(REPS + 2):
    st = {}
    for name, fn in stages:
        t0 = time.perf_counter()
        fn(st)
        if it >= 2:
            acc[name] += time.perf_counter() - t0
print("reference", {n: round(v / REPS * 1e3, 2) for n, v in acc.items()})

O.build()
fs, c = a.sampling_frequency, p.sound_speed
ol = O.kk_luts(g.x, g.z, p.transmit_angles, rx.angles, c)
ones = np.ones(rx.num_angles)
shift = -p.start_time * fs
tr = O.decompose_c64_staged(rfa, fs, a.positions, rx.angles, c)
O.kk_kernel(tr, *ol, ones, fs, shift)


def t(fn):
    fn()
    t0 = time.perf_counter()
    for _ in range(REPS):
        fn()
    return round((time.perf_counter() - t0) / REPS * 1e3, 2)


print("port", {"stage1": t(lambda: O.decompose_c64_staged(rfa, fs, a.positions, rx.angles, c)),
               "kk": t(lambda: O.kk_kernel(tr, *ol, ones, fs, shift)),
               "db": t(lambda: O.log_compress_db(O.intensity(tr[0, :1, :1])))})
