"""Per-frame latency of the drop-in path (numpy in, numpy out), configs 1 and 4.

What an unmodified kkbeam caller gets:
* ``kk_kernel``: the shim the reference's ``kk`` calls once ``kkbeam_plugin``
  is installed (beamform.py:363-374): complex64 traces + four float64 tables
  in, complex128 image out, with the plan cached across calls on the same
  tables;
* ``kk``: this package's ``kk(CompressedRF, DelayLUTSet)`` (same signature
  as the reference's, container validation included);
* ``pipeline``: ``analytic_signal -> compress -> kk`` through the public API,
  numpy at every boundary (the reference's README flow).
Beside them, on the same host: the oracle's C/OpenMP restatement of
``_kk_kernel`` (all cores) and the reference benchmark's complex64 stage 1
(numpy/scipy) — the CPU cost each call replaces.

Median of 30 calls after 5 warm-ups, host wall clock (time.perf_counter):
these are host-API latencies, including the H2D / D2H copies.
usage: python scripts/dropin_latency.py [out.json]
"""

from __future__ import annotations

import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def med(fn, reps=30, warm=5):
    for _ in range(warm):
        fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    return 1e3 * statistics.median(t)


def main():
    import paper_2603_22496_b200 as kb
    from oracle import kkbeam_oracle as O
    from paper_2603_22496_b200 import configs, kkbeam_plugin
    from paper_2603_22496_b200.beamform import kk_plans

    O.build()
    res = {"tool": "scripts/dropin_latency.py", "unit": "ms per frame (median, host wall clock)",
           "cpu_threads": os.cpu_count(), "configs": {}}
    for cfg in (1, 4):
        w = configs.CONFIGS[cfg]() if cfg == 1 else configs.config4(frames=1)
        arr, p, rx, g = w.array, w.params, w.receive, w.grid
        fs, c = arr.sampling_frequency, p.sound_speed
        rf = configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=3)
        tr = O.decompose_c64_staged(rf, fs, arr.positions, rx.angles, c)
        luts = O.kk_luts(g.x, g.z, p.transmit_angles, rx.angles, c)
        ones = np.ones(rx.num_angles)
        shift = (0.0 - p.start_time) * fs
        out = np.empty((g.nx, g.nz), np.complex128)
        r = {}
        r["kk_kernel_shim_gpu"] = med(lambda: kkbeam_plugin.kk_kernel(tr, *luts, ones, fs, shift, True, out))
        ref = O.kk_kernel(tr, *luts, ones, fs, shift)
        r["kk_kernel_shim_rel_l2_vs_oracle"] = float(np.linalg.norm(out - ref) / np.linalg.norm(ref))
        r["kk_kernel_oracle_cpu_all_cores"] = med(lambda: O.kk_kernel(tr, *luts, ones, fs, shift), reps=10)
        an = kb.analytic_signal(kb.RFVolume(rf, arr, p))
        rfc = kb.compress(an, rx)
        dl = kb.build_kk_luts(g, p, rx)
        r["kk_api_gpu"] = med(lambda: kb.kk(rfc, dl))
        r["pipeline_api_gpu"] = med(lambda: kb.kk(kb.compress(kb.analytic_signal(kb.RFVolume(rf, arr, p)), rx), dl))
        r["stage1_reference_form_cpu"] = med(lambda: O.decompose_c64_staged(rf, fs, arr.positions, rx.angles, c),
                                             reps=10)
        r["plan_cache"] = {"hits": kk_plans.hits, "misses": kk_plans.misses}
        r["pixel_pairs"] = g.nx * g.nz * w.pairs
        res["configs"][w.name] = r
        print(w.name, json.dumps(r), flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
