"""Per-frame latency of the drop-in path (numpy in, numpy out), configs 1 and 4.

What an unmodified kkbeam caller gets:
* ``kk_kernel``: the shim the reference's ``kk`` calls once ``kkbeam_plugin``
  is installed (beamform.py:363-374): complex64 traces + four float64 tables
  in, complex128 image out, with the plan cached across calls on the same
  tables;
* ``kk``: this package's ``kk(CompressedRF, DelayLUTSet)`` (same signature
  as the reference's, container validation included);
* ``pipeline``: ``analytic_signal -> compress -> kk`` through the public API,
  numpy at every boundary (the reference's README flow);
* with the reference installed in baseline/_ref: its own README pipeline,
  unmodified, on the host (numba / numpy) and with ``kkbeam_plugin``
  installed (its kernels and analytic_signal rebound to libkkb).
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
    # the unmodified reference's README pipeline, numba/numpy on the host vs
    # the same calls with kkbeam_plugin installed (when baseline/_ref holds it)
    ref_root = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref_root, "kkbeam")):
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_dropin")
        sys.path.insert(0, ref_root)
        import kkbeam as rk

        for cfg in (1, 4):
            w = configs.CONFIGS[cfg]() if cfg == 1 else configs.config4(frames=1)
            arr, p, rx, g = w.array, w.params, w.receive, w.grid
            rarr = rk.TransducerArray(arr.num_elements, arr.pitch, arr.center_frequency,
                                      arr.sampling_frequency, arr.fractional_bandwidth)
            rp = rk.AcquisitionParams(p.sound_speed, p.transmit_angles, p.num_samples, start_time=p.start_time)
            rrx = rk.explicit_angles(rx.angles, rx.delta_theta_i)
            rg = rk.ImageGrid(g.x0, g.z0, g.dx, g.dz, g.nx, g.nz)
            rf = rk.RFVolume(configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=3), rarr, rp)
            luts = rk.build_kk_luts(rg, rp, rrx)

            def pipe():
                return rk.kk(rk.compress(rk.analytic_signal(rf), rrx), luts)

            cpu_ms = med(pipe, reps=5, warm=3)
            cpu_img = pipe().pixels
            h = kkbeam_plugin.install(rk)
            try:
                gpu_ms = med(pipe, reps=20, warm=3)
                gpu_img = pipe().pixels
            finally:
                h.restore()
            r = {"reference_pipeline_cpu_ms": cpu_ms, "reference_pipeline_with_plugin_ms": gpu_ms,
                 "speedup": cpu_ms / gpu_ms,
                 "rel_l2_plugin_vs_cpu": float(np.linalg.norm(gpu_img - cpu_img) / np.linalg.norm(cpu_img))}
            res["configs"][w.name]["unmodified_reference_readme_pipeline"] = r
            print(w.name, "reference pipeline", json.dumps(r), flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
