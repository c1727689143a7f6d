"""The reference's staged benchmark (kkbeam.bench.bench_kk / bench_das,
bench.py:156-185) on its own CPU stages and, through kkbeam_plugin, on the
GPU stages (paper_2603_22496_b200.bench): per-stage medians for config 1 and
config 4 geometries on the reference's seeded noise volume.
usage: PYTHONPATH=baseline/_ref:. python scripts/staged_bench.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_staged")


def main():
    import kkbeam as rk

    from paper_2603_22496_b200 import configs, kkbeam_plugin

    res = {"tool": "scripts/staged_bench.py", "unit": "ms per stage (median of 3 after a discarded run, "
           "host wall clock; GPU stages end with a device sync)", "rows": []}
    for name, w in (("config1", configs.config1()), ("config4", configs.config4(frames=1))):
        a, p, rx, g = w.array, w.params, w.receive, w.grid
        arr = rk.TransducerArray(a.num_elements, a.pitch, a.center_frequency, a.sampling_frequency,
                                 a.fractional_bandwidth)
        par = rk.AcquisitionParams(p.sound_speed, p.transmit_angles, p.num_samples, start_time=p.start_time)
        rrx = rk.explicit_angles(rx.angles, rx.delta_theta_i)
        grid = rk.ImageGrid(g.x0, g.z0, g.dx, g.dz, g.nx, g.nz)
        rf = rk.noise_volume(arr, par, seed=0)
        for side in ("cpu", "gpu"):
            h = kkbeam_plugin.install(rk) if side == "gpu" else None
            try:
                rows = [rk.bench_kk(rf, grid, rrx, 3), rk.bench_das(rf, grid, 3)]
            finally:
                if h:
                    h.restore()
            for r in rows:
                rec = {"config": name, "side": side, "label": r.label,
                       **{s + "_ms": r.stage_ms(s) for s in rk.bench.STAGES}, "total_ms": r.total_ms}
                res["rows"].append(rec)
                print(json.dumps(rec), flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
