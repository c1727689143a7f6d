"""Golden outputs of the reference's staged-benchmark helpers (kkbeam/bench.py:
noise_volume, write_bench_csv, format_bench_table) for tests/test_bench_api.py.

Run in the build container, where the reference is importable:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bench_golden.py
Writes tests/golden/bench.npz (small: a checksum of the noise volume and the
two text renderings of two fixed rows)."""
import hashlib
import os

import numpy as np

import kkbeam as rk

arr = rk.TransducerArray(16, 0.3e-3, 5.0e6, 20.0e6, 0.6)
par = rk.AcquisitionParams(1540.0, np.array([-0.1, 0.0, 0.1]), 256)
vol = rk.noise_volume(arr, par, seed=7)
rows = [rk.StageTimings("kk_m5", "kk", 5, 16 / 5, 1234, 1.25, 2.5, 0.125, 3.0),
        rk.StageTimings("das", "das", 16, 1.0, 98765, 10.0, 0.5, 7.75, 20.0)]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bench.npz")
np.savez(out, volume_sha=hashlib.sha256(vol.data.tobytes()).hexdigest(), volume_shape=np.array(vol.data.shape),
         csv=rk.bench_csv_text(rows), table=rk.format_bench_table(rows))
print("wrote", out)
