"""KKRF ingest rate: config-4 frames stored one per KKRF
file, read straight into HBM by the native pinned double-buffered reader
(rffile.read_ensemble_device), then the whole hot path on them.  Files live
in /tmp on the box (page-cache warm after the write, so this is the
host-memory -> HBM leg, the ceiling of any disk)."""
import json
import os
import shutil
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import configs, rffile  # noqa: E402

F = 64
w = configs.config4(frames=F)
a, p = w.array, w.params
d = tempfile.mkdtemp(prefix="kkrf_")
try:
    paths = []
    for f in range(F):
        rf = kb.RFVolume(configs.noise_rf(p.num_transmits, a.num_elements, p.num_samples, seed=f), a, p)
        path = os.path.join(d, f"frame{f:03d}.rf")
        rffile.write_container(path, rf)
        paths.append(path)
    reps = 3
    sweep = {}
    for th in (1, 2, 4, 8, 16):
        t, meta = rffile.read_ensemble_device(paths, threads=th)  # warm (slots, page cache)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            t, meta = rffile.read_ensemble_device(paths, threads=th)
        torch.cuda.synchronize()
        sweep[th] = (time.perf_counter() - t0) / reps
    nbytes = t.numel() * t.element_size()
    dt = sweep[8]
    eng = kb.KKEngine(a, p, w.receive, w.grid, frames=F)
    eng.run(t)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        t, meta = rffile.read_ensemble_device(paths)
        eng.run(t)
    torch.cuda.synchronize()
    dt2 = (time.perf_counter() - t0) / reps
    ok = bool(torch.equal(t[5].cpu(), torch.from_numpy(configs.noise_rf(p.num_transmits, a.num_elements,
                                                                        p.num_samples, seed=5))))
    print(json.dumps({"frames": F, "bytes": nbytes,
                      "read_GBps_by_threads": {k: nbytes / v / 1e9 for k, v in sweep.items()},
                      "read_GBps": nbytes / dt / 1e9,
                      "read_ms_per_frame": dt / F * 1e3,
                      "read_plus_beamform_frames_per_s": F / dt2, "payload_exact": ok}))
    eng.close()
finally:
    shutil.rmtree(d, ignore_errors=True)
