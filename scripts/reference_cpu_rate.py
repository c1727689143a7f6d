"""The reference itself (kkbeam from the git-ignored baseline/_ref, numba on
all host cores) on one config-4 frame, next to the oracle port that bench.py's
cpu_baseline / --impl reference arm times: validates that the port is a fair
stand-in for the reference's CPU path.  Stages are the reference benchmark's
own (bench.py:113-153: scipy FFT, weighted einsum per receive angle, IFFT,
then kk)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(1, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import numpy as np  # noqa: E402

import kkbeam as R  # noqa: E402  (the reference package)
from kkbeam import bench as RB  # noqa: E402

from paper_2603_22496_b200 import configs  # noqa: E402

w = configs.config4(frames=1)
g, a, p, rx = w.grid, w.array, w.params, w.receive
arr = R.TransducerArray(a.num_elements, a.pitch, a.center_frequency, a.sampling_frequency,
                        a.fractional_bandwidth)
params = R.AcquisitionParams(p.sound_speed, np.asarray(p.transmit_angles), p.num_samples,
                             start_time=p.start_time)
recv = R.uniform_vernier_angles(11, 11, 10 * np.pi / 180, 0)
assert np.array_equal(recv.angles, rx.angles)
grid = R.ImageGrid(g.x0, g.z0, g.dx, g.dz, g.nx, g.nz)
rf = R.RFVolume(configs.noise_rf(p.num_transmits, a.num_elements, p.num_samples, seed=0), arr, params)
luts = R.build_kk_luts(grid, params, recv)
stages = RB._kk_stage_fns(rf, recv, luts, R.BeamformConfig())


def frame():
    st = {}
    for _, fn in stages:
        fn(st)
    return st


frame()  # numba compile, scipy plans
n, t0 = 0, time.perf_counter()
while n < 3 or time.perf_counter() - t0 < 10.0:
    frame()
    n += 1
ref_ms = (time.perf_counter() - t0) / n * 1e3

sys.path.insert(0, ROOT)
import bench  # noqa: E402

rate, m, dt = bench.cpu_pipeline_rate(w, seconds=10.0, min_frames=3)
print(json.dumps({"workload": w.name, "frame": "one config-4 frame (11 x 11 pairs, 256 x 256 px, T=1536)",
                  "reference_ms_per_frame": ref_ms, "reference_frames": n,
                  "port_ms_per_frame": 1e3 / rate, "port_frames": m,
                  "host_cores": os.cpu_count(),
                  "note": "reference: its own bench stages (scipy + numba kk on all cores); "
                          "port: oracle/ numpy stage 1 + C/OpenMP kk + intensity/dB"}))
